"""GPU parity of the separable 2D SL kernel (step2d.cu sl2d_sep_kernel).

BASELINE's 2D speed traces departures whose x-record does not depend on the
mesh row and whose y-record does not depend on the column, so the fine-level
SL step runs the sliding-window kernel.  Its rows must be bit-identical to the
reference's tensor-product gather (semi_lagrangian.py:238-253, restated in
oracle.sl_apply) for every strip height, across the periodic wrap in both
directions, for coarse (large-CFL) plain-SL levels whose window advances by
0, 1 or several source rows per mesh row (tiles whose source window does not
fit the staged tile gather per node), and in every output form.  The kernel
reads only one x-record per column and one y-record per row and trusts the
level's hint, so the hint's detection is tested to be exact.
"""

import os

import numpy as np
import pytest
import torch

import oracle as O
from test_gpu_production2d import _np, _oracle_level

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import paper_2203_13382_b200 as P
    assert torch.cuda.is_available(), "GPU tests need CUDA"
    return P


@pytest.fixture
def sep_rows():
    """Set the strip height of the kernel for one test (restored afterwards)."""
    prev = os.environ.get("MGRIT_SL2D_SEP_ROWS")

    def set_rows(nb):
        if nb is None:
            os.environ.pop("MGRIT_SL2D_SEP_ROWS", None)
        else:
            os.environ["MGRIT_SL2D_SEP_ROWS"] = str(nb)
    yield set_rows
    set_rows(int(prev) if prev is not None else None)


def _levels(P, n_x, p, n_t=16, m=4, **kw):
    cfg = P.SolverConfig(n_x=n_x, n_t=n_t, dim=2, wave_speed="B4", p=p, schedule=m, seed=3, u0="sin4", **kw)
    return P.build_hierarchy(cfg)


@pytest.mark.parametrize("p", [1, 3, 5])
@pytest.mark.parametrize("nb", [8, 16, 32, None])
def test_sep_fine_rows_bitwise(P, sep_rows, p, nb):
    """Fine SL rows on a 256^2 mesh (every CTA touches the x-wrap, two bands
    touch the y-wrap), every strip height; 0 = the column-strip kernel."""
    fine = _levels(P, 256, p)[0]
    assert fine.separable
    steps = [0, 5, 11, 15]
    ol = _oracle_level(fine, steps)
    U = np.random.default_rng(100 + p).standard_normal((len(steps), fine.grid.n_points))
    Ud = torch.from_numpy(U).cuda()
    sep_rows(nb)
    got = _np(fine.step_batch(np.array(steps), Ud))
    sep_rows(0)
    strip = _np(fine.step_batch(np.array(steps), Ud))
    for b, t in enumerate(steps):
        want = ol.step(t, U[b])
        assert np.array_equal(got[b], want), (p, nb, t)
        assert np.array_equal(strip[b], want), (p, "strip", t)


@pytest.mark.parametrize("p", [3, 5])
def test_sep_large_cfl_levels_bitwise(P, sep_rows, p):
    """Plain-SL coarse levels traced with the coarse step (erk_rediscretized):
    the y-window advances by 0, 1 or several source rows per mesh row."""
    levels = _levels(P, 256, p, n_t=64, m=4, operator_kind="rediscretized", departure_policy="erk_rediscretized")
    for lv in levels[1:]:
        assert lv.separable, lv.index
        steps = list(range(min(lv.n_steps, 3)))
        ol = _oracle_level(lv, steps)
        U = np.random.default_rng(7 + lv.index).standard_normal((len(steps), lv.grid.n_points))
        for nb in (8, 32):
            sep_rows(nb)
            got = _np(lv.step_batch(np.array(steps), torch.from_numpy(U).cuda()))
            for b, t in enumerate(steps):
                assert np.array_equal(got[b], ol.step(t, U[b])), (p, lv.index, nb, t)
        # the window really moves by other amounts than one row on this level
        ey = np.ceil(_np(lv.s_y[0]).reshape(256, 256)[:, 0]).astype(np.int64)
        d = np.diff(ey) % 256
        if lv.index == len(levels) - 1:
            assert (d != 1).any()


def _separable_flag(P, lv):
    from paper_2203_13382_b200 import _lib
    from paper_2203_13382_b200.mgrit import stream_ptr
    flag = torch.full((1,), -7, dtype=torch.int32, device="cuda")
    rc = _lib.load().mgrit_records_separable(lv.grid.n_x, lv.s_x.shape[0], lv.s_x.data_ptr(), lv.s_y.data_ptr(),
                                             flag.data_ptr(), stream_ptr())
    assert rc == 0
    return int(flag.item())


def test_separable_hint_detection(P):
    """The kernel trusts the hint, so the hint must be exact: it is computed
    over every record of the level (mgrit_records_separable), says no for a
    speed whose x-component depends on y (C5), and says no when a single
    record of a separable level is one ulp off."""
    cfg = P.SolverConfig(n_x=256, n_t=8, dim=2, wave_speed="C5", p=3, schedule=4, seed=1)
    c5 = P.build_hierarchy(cfg)[0]
    assert not c5.separable and _separable_flag(P, c5) == 0
    # ... and the non-separable level runs the generic kernels, bit-identical
    steps = [0, 3, 7]
    ol = _oracle_level(c5, steps)
    U = np.random.default_rng(5).standard_normal((len(steps), c5.grid.n_points))
    got = _np(c5.step_batch(np.array(steps), torch.from_numpy(U).cuda()))
    for b, t in enumerate(steps):
        assert np.array_equal(got[b], ol.step(t, U[b])), t

    fine = _levels(P, 256, 5)[0]
    assert fine.separable and _separable_flag(P, fine) == 1
    for arr, idx in ((fine.s_y, 77 * 256 + 130), (fine.s_x, 255 * 256 + 255), (fine.s_x, 1 * 256 + 0)):
        keep = arr[2, idx].item()
        arr[2, idx] = np.nextafter(keep, 1e9)
        try:
            assert _separable_flag(P, fine) == 0
        finally:
            arr[2, idx] = keep
    assert _separable_flag(P, fine) == 1
    # every coarse level of the BASELINE hierarchy is checked on its own
    for lv in _levels(P, 256, 3, n_t=64, m=4)[1:]:
        assert lv.separable == bool(_separable_flag(P, lv))


@pytest.mark.parametrize("nb", [8, 32, None])
def test_sep_output_forms_and_row_norms(P, sep_rows, nb):
    """S u + g, g + S u - v (residual form) and the per-row sums of squares;
    the sums do not depend on the strip height."""
    fine = _levels(P, 256, 3)[0]
    n = fine.grid.n_points
    steps = [1, 4, 9]
    B = len(steps)
    ol = _oracle_level(fine, steps)
    rng = np.random.default_rng(21)
    U, G, V = (rng.standard_normal((B, n)) for _ in range(3))
    Ud, Gd, Vd = (torch.from_numpy(x).cuda() for x in (U, G, V))
    t_idx = torch.as_tensor(steps, device="cuda")
    sep_rows(nb)
    out = torch.empty((B, n), dtype=torch.float64, device="cuda")
    ss = torch.zeros(B, dtype=torch.float64, device="cuda")
    fine._apply(Ud, 0, 0, B, out, G=Gd, t_idx=t_idx, row_sumsq=ss)
    for b, t in enumerate(steps):
        want = ol.step(t, U[b]) + G[b]
        assert np.array_equal(_np(out[b]), want)
        assert abs(ss[b].item() - np.sum(want * want)) <= 1e-13 * np.sum(want * want)
    ss1 = ss.clone()
    fine._apply(Ud, 0, 0, B, out, G=Gd, U_sub=Vd, t_idx=t_idx, row_sumsq=ss)
    for b, t in enumerate(steps):
        want = (G[b] + ol.step(t, U[b])) - V[b]
        assert np.array_equal(_np(out[b]), want)
    # norms only (no output row)
    ss2 = torch.zeros(B, dtype=torch.float64, device="cuda")
    fine._apply(Ud, 0, 0, B, None, G=Gd, t_idx=t_idx, row_sumsq=ss2)
    assert torch.equal(ss1, ss2)
    sep_rows(8)
    ss3 = torch.zeros(B, dtype=torch.float64, device="cuda")
    fine._apply(Ud, 0, 0, B, None, G=Gd, t_idx=t_idx, row_sumsq=ss3)
    assert torch.equal(ss1, ss3), "row norms must not depend on the strip height"


def test_sep_production_meshes_bitwise(P, sep_rows):
    """cfg4's and cfg5's meshes/degrees through the kernel at its default strip height."""
    for n_x, p in ((512, 3), (1024, 5)):
        fine = _levels(P, n_x, p, n_t=8, m=4)[0]
        assert fine.separable
        steps = [0, 7]
        ol = _oracle_level(fine, steps)
        U = np.random.default_rng(n_x).standard_normal((2, fine.grid.n_points))
        got = _np(fine.step_batch(np.array(steps), torch.from_numpy(U).cuda()))
        for b, t in enumerate(steps):
            assert np.array_equal(got[b], ol.step(t, U[b])), (n_x, t)


@pytest.mark.parametrize("kw", [
    dict(n_x=256, n_t=64, dim=2, wave_speed="B4", p=3, schedule=4, seed=3, u0="sin4"),
    dict(n_x=4096, n_t=256, wave_speed="B2", p=3, schedule=4, seed=1),
    dict(n_x=16384, n_t=128, wave_speed="B2", p=5, schedule=8, seed=2),
    dict(n_x=1024, n_t=128, wave_speed="C1", p=1, schedule=8, max_levels=2, dt=0.85 * 2.0 / 1024),
], ids=["2d", "1d_n4096", "1d_n16384", "1d_two_level"])
def test_fine_fc_phase_skips_redundant_f_relaxation_bitwise(P, kw):
    """Solves run the fine FC phase without its F-steps (the previous
    V-cycle's closing F-relaxation, mgrit.py:334, already produced those
    rows; _FusedCycle.prologue covers the first cycle): 2D through
    mgrit_phase_args::f_relaxed, 1D as one batched row launch.  Iterates and
    histories are bit-identical to the engine that repeats them."""
    from paper_2203_13382_b200 import _lib, mgrit as M
    kw = dict(kw, max_iters=4, rtol=0.0)
    cfg = P.SolverConfig(**kw)
    levels = P.build_hierarchy(cfg)
    outs = []
    for skip in (True, False):
        levels[0].__dict__.pop("_sessions", None)
        sess = M._session(levels, cfg, torch.device("cuda"))
        assert sess.engine.skip_f
        if not skip:
            sess.engine.skip_f = False
            sess.engine._args[(0, _lib.PHASE_FC)].f_relaxed = 0
        rep, U = P.solve(cfg, levels, output="device", use_graph=skip)
        outs.append((rep.residual_norms.copy(), U.clone()))
    levels[0].__dict__.pop("_sessions", None)
    assert np.array_equal(outs[0][0], outs[1][0])
    assert torch.equal(outs[0][1], outs[1][1])
