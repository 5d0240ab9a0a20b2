"""Host-side logic of the operator-level API (no GPU): argument validation and
error behaviour mirror the reference (semi_lagrangian.py:21-72,
coarse_correction.py:35-47, 69-89, 173-182)."""

import numpy as np
import pytest

import oracle as O
import paper_2203_13382_b200 as P


def test_stencil_extents_and_degree_errors():
    assert P.stencil_extents(1) == (1, 0) and P.stencil_extents(3) == (2, 1) and P.stencil_extents(5) == (3, 2)
    for bad in (0, 2, 7):
        with pytest.raises(ValueError):
            P.stencil_extents(bad)
        with pytest.raises(ValueError):
            P.derivative_stencil(bad)


@pytest.mark.parametrize("order", [1, 3, 5])
def test_erk_scheme_constants(order):
    s = P.erk_scheme(order)
    a, b, c = O.erk_tableau(order)
    assert s.n_stages == len(b)
    assert np.array_equal(s.a, a) and np.array_equal(s.b, b) and np.array_equal(s.c, c)
    with pytest.raises(ValueError):
        P.erk_scheme(2)


def test_derivative_stencils_match_reference():
    for p in (1, 3, 5):
        assert np.array_equal(P.derivative_stencil(p), O.d_stencil(p))


def test_correction_field_add():
    a = P.CorrectionField(np.ones(4))
    b = P.CorrectionField(np.full(4, 2.0))
    assert np.array_equal((a + b).x, np.full(4, 3.0)) and (a + b).dim == 1
    with pytest.raises(ValueError):
        a + P.CorrectionField(np.ones(4), np.ones(4))


def test_gmres_solve_rejects_host_callables():
    """No CPU fallback: an arbitrary Python operator has no device form."""
    with pytest.raises(TypeError):
        P.gmres_solve(lambda v: v, np.ones(8), P.GmresConfig(10, None))


def test_apply_imsd_needs_a_derivative_stencil():
    from paper_2203_13382_b200.operators import _degree_of_stencil
    assert _degree_of_stencil(P.derivative_stencil(3)) == 3
    with pytest.raises(ValueError):
        _degree_of_stencil(np.array([1.0, -3.0, 1.0]))
