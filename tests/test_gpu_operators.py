"""The operator-level drop-in API below Level (mgrit_advect/__init__.py:8-16)
against the REAL reference's golden vectors (tests/golden/ops.npz, made by
make_golden.py from mgrit_advect) and the oracle:

* decompose, interp_weights, sl_step (fed the reference's own DepartureSets
  through the records-from-(east, eps) entry) and apply_ImSD: bit-identical;
* gmres_solve (fixed and tolerance mode) and corrected_coarse_step: solution
  within 1e-13 relative, the residual history within 1e-12 relative and of
  identical length (the iteration count);
* forward_euler_coarse_step: bit-identical;
* Level views (departures / sigma / dep / sig / _idx / _w) equal the oracle
  hierarchy's records bit-for-bit.
"""

import numpy as np
import pytest
import torch

import oracle as O
from oracle import mgrit_oracle as OM

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import paper_2203_13382_b200 as P
    assert torch.cuda.is_available()
    return P


def _np(t):
    return t.detach().cpu().numpy() if isinstance(t, torch.Tensor) else np.asarray(t)


@pytest.mark.parametrize("n", [16, 64, 1024])
def test_decompose_bitwise(P, ops, n):
    east, eps = P.decompose(P.Grid1D(n), ops[f"dec_n{n}_coords"])
    assert np.array_equal(east, ops[f"dec_n{n}_east"])
    assert np.array_equal(eps, ops[f"dec_n{n}_eps"])
    # device tensors in, device tensors out
    e2, x2 = P.decompose(P.Grid1D(n), torch.as_tensor(ops[f"dec_n{n}_coords"]).cuda())
    assert e2.is_cuda and np.array_equal(_np(e2), east) and np.array_equal(_np(x2), eps)


@pytest.mark.parametrize("p", [1, 3, 5])
def test_interp_weights_bitwise(P, ops, p):
    assert np.array_equal(P.interp_weights(p, ops[f"w_p{p}_eps"]), ops[f"w_p{p}"])


def _refdep(P, ops, key, dim):
    """The reference's DepartureSet of an ops.npz ERK case (east/eps only)."""
    e, x = ops[key + "_east"], ops[key + "_eps"]
    if dim == 1:
        return P.DepartureSet1D(0.37, 0.1, e, x, ops[key + "_disp"])
    return P.DepartureSet2D(0.37, 0.1, e[0], e[1], x[0], x[1], ops[key + "_disp"][0], ops[key + "_disp"][1])


SL_CASES = [("C1", 1, 64), ("C2", 1, 64), ("C3", 1, 64), ("B2", 1, 128), ("C4", 2, 16), ("C5", 2, 16),
            ("B4", 2, 24)]


@pytest.mark.parametrize("speed,dim,n", SL_CASES)
@pytest.mark.parametrize("order", [1, 3, 5])
def test_sl_step_from_reference_departure_sets_bitwise(P, ops, speed, dim, n, order):
    """sl_step(grid, <the reference's DepartureSet>, p, u) == the reference's
    sl_step output, bit for bit, for p = 1, 3, 5."""
    key = f"erk_{speed}_r{order}"
    grid = P.Grid1D(n) if dim == 1 else P.Grid2D(n)
    dep = _refdep(P, ops, key, dim)
    u = ops[key + "_u"]
    for p in (1, 3, 5):
        assert np.array_equal(P.sl_step(grid, dep, p, u), ops[key + f"_sl_p{p}"]), (key, p)


GM_CASES = [(d, n, p, s) for d, n in ((1, 64), (1, 256), (2, 16)) for p in (1, 3, 5) for s in (0.0, 0.05, 0.6)]


def _field(P, ops, key, dim):
    return P.CorrectionField(ops[key + "_sx"], ops[key + "_sy"] if dim == 2 else None)


@pytest.mark.parametrize("dim,n,p,scale", GM_CASES)
def test_apply_ImSD_bitwise(P, ops, dim, n, p, scale):
    key = f"gm_d{dim}_n{n}_p{p}_s{scale}"
    grid = P.Grid1D(n) if dim == 1 else P.Grid2D(n)
    got = P.apply_ImSD(_field(P, ops, key, dim), P.derivative_stencil(p), ops[key + "_rhs"], grid)
    assert np.array_equal(got, ops[key + "_imsd"])


@pytest.mark.parametrize("dim,n,p,scale", GM_CASES)
@pytest.mark.parametrize("mode", ["fixed", "tol"])
def test_gmres_solve_matches_reference(P, ops, dim, n, p, scale, mode):
    key = f"gm_d{dim}_n{n}_p{p}_s{scale}"
    grid = P.Grid1D(n) if dim == 1 else P.Grid2D(n)
    op = P.ImSD(_field(P, ops, key, dim), P.derivative_stencil(p), grid)
    cfg = P.GmresConfig(10, None if mode == "fixed" else 1e-2)
    x, hist = P.gmres_solve(op, ops[key + "_rhs"], cfg)
    want_x, want_h = ops[key + f"_{mode}_x"], ops[key + f"_{mode}_hist"]
    assert len(hist) == len(want_h)                      # the iteration count
    # |g_k| differences relative to beta (the solve-history bar: late entries
    # are tiny and carry the reductions' rounding relative to beta, not to themselves)
    assert np.max(np.abs(hist - want_h)) <= 1e-12 * want_h[0]
    assert np.linalg.norm(x - want_x) <= 1e-13 * max(np.linalg.norm(want_x), 1e-300)


def test_gmres_solve_errors(P):
    g = P.Grid1D(16)
    op = P.ImSD(P.CorrectionField(np.full(16, 0.1)), P.derivative_stencil(1), g)
    x, h = P.gmres_solve(op, np.zeros(16), P.GmresConfig(10, 1e-2))
    assert np.array_equal(x, np.zeros(16)) and list(h) == [0.0]
    bad = np.ones(16)
    bad[2] = np.inf
    with pytest.raises(ValueError):
        P.gmres_solve(op, bad, P.GmresConfig(10, None))
    with pytest.raises(TypeError):
        P.gmres_solve(lambda v: v, np.ones(16), P.GmresConfig(10, None))


@pytest.mark.parametrize("dim,n,speed", [(1, 128, "B2"), (2, 24, "B4")])
@pytest.mark.parametrize("p", [1, 3, 5])
def test_coarse_steps_match_oracle(P, dim, n, speed, p):
    """corrected_coarse_step (1e-13) and forward_euler_coarse_step (bitwise)
    on a backtracked coarse DepartureSet and its sigma, from the oracle."""
    kw = dict(n_x=n, n_t=16, dim=dim, wave_speed=speed, p=p, schedule=4, max_levels=2)
    olv = O.hierarchy(O.OConfig(**kw))[1]
    od, sig = olv.deps[2], olv.sigma[2]
    grid = P.Grid1D(n) if dim == 1 else P.Grid2D(n)
    if dim == 1:
        dep = P.DepartureSet1D(0.0, olv.dt, od.east[0], od.eps[0], None)
        field = P.CorrectionField(sig[0])
    else:
        dep = P.DepartureSet2D(0.0, olv.dt, od.east[0], od.east[1], od.eps[0], od.eps[1], None, None)
        field = P.CorrectionField(sig[0], sig[1])
    u = np.random.default_rng(p).standard_normal(grid.n_points)
    for tol in (None, 1e-2):
        got = P.corrected_coarse_step(grid, dep, p, field, P.GmresConfig(10, tol), u)
        want, _ = O.gmres(lambda v: O.imsd(sig, O.d_stencil(p), v, n), O.sl_apply(dim, n, p, od, u), 10, tol)
        assert np.linalg.norm(got - want) <= 1e-13 * np.linalg.norm(want)
    fe = P.forward_euler_coarse_step(grid, dep, p, field, u)
    assert np.array_equal(fe, OM.ipsd(sig, O.d_stencil(p), O.sl_apply(dim, n, p, od, u), n))


def test_level_views_match_oracle_records(P):
    """Level.departures / sigma / dep(n) / sig(n) / _idx / _w (mgrit.py:89-126)."""
    for kw in (dict(n_x=64, n_t=128, wave_speed="B2", p=5, schedule=8),
               dict(n_x=16, n_t=64, dim=2, wave_speed="C5", p=3, schedule=4)):
        ocfg = O.OConfig(**kw)
        olevels = O.hierarchy(ocfg)
        fine = olevels[0]
        coords = (np.stack([d.coords[0] for d in fine.deps]) if fine.dim == 1 else
                  (np.stack([d.coords[0] for d in fine.deps]), np.stack([d.coords[1] for d in fine.deps])))
        levels = P.build_hierarchy(P.SolverConfig(**kw), fine_coords=coords)
        for lv, ol in zip(levels, olevels):
            assert len(lv.departures) == len(ol.deps)
            for n in (0, lv.n_steps - 1):
                d, od = lv.dep(n), ol.dep(n)
                if lv.grid.dim == 1:
                    assert np.array_equal(_np(d.east), od.east[0]) and np.array_equal(_np(d.eps), od.eps[0])
                else:
                    assert np.array_equal(_np(d.east_x), od.east[0]) and np.array_equal(_np(d.nu), od.eps[1])
                if ol.sigma is not None:
                    assert np.array_equal(_np(lv.sig(n).x), ol.sig(n)[0])
            if lv.grid.dim == 1:
                ell, r = OM.extents(lv.p)
                want_idx = np.stack([np.stack([np.mod(d.east[0] + j, lv.grid.n_x) for j in range(-ell, r + 1)], 1)
                                     for d in ol.deps])
                assert np.array_equal(_np(lv._idx), want_idx)
                assert np.array_equal(_np(lv._w), np.stack([O.lagrange_weights(lv.p, d.eps[0]) for d in ol.deps]))
    # constant speed: one shared set (reference test_mgrit.py:188-194)
    levels = P.build_hierarchy(P.SolverConfig(n_x=32, n_t=64, wave_speed="C1", p=1, schedule=4))
    assert levels[0].shared and len(levels[0].departures) == 1
    levels = P.build_hierarchy(P.SolverConfig(n_x=32, n_t=64, wave_speed="C2", p=1, schedule=4))
    assert not levels[0].shared and len(levels[0].departures) == 64
