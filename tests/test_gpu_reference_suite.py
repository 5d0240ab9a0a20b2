"""GPU ports of the reference's own hot-path unit tests (pkg/tests/
test_semi_lagrangian.py, test_coarse_correction.py, test_mgrit.py), run against
the CUDA operators through the drop-in API.  Each test cites the reference
test it mirrors."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import paper_2203_13382_b200 as P
    assert torch.cuda.is_available()
    return P


def _np(t):
    return t.detach().cpu().numpy()


def sl_level(grid, coords, p, kind="fine", sig=None, gmres=None):
    """A one-step level from caller departure coordinates (shared record)."""
    from paper_2203_13382_b200 import mgrit as M
    s_x, s_y, _, _ = M.departures_from_coords(grid, coords)
    lv = M.Level(0, grid, p, 1, 0.1, kind, s_x[:1], None if s_y is None else s_y[:1], shared=True)
    if sig is not None:
        sx = sig[0] if grid.dim == 2 else sig
        lv.sig_x = torch.as_tensor(np.asarray(sx, dtype=np.float64)).reshape(1, -1).cuda()
        if grid.dim == 2:
            lv.sig_y = torch.as_tensor(np.asarray(sig[1], dtype=np.float64)).reshape(1, -1).cuda()
    lv.gmres_cfg = gmres
    return lv


def step(lv, u):
    return _np(lv.step(0, torch.as_tensor(np.asarray(u, dtype=np.float64)).cuda()))


# ---- test_semi_lagrangian.py ------------------------------------------------


def test_sl_nodal_departures_copy_state(P):
    """eps = 0 (departure on a node) is an exact copy (test_interp_weights_nodal :82-89)."""
    g = P.Grid1D(32)
    u = np.random.default_rng(0).random(32)
    for p in (1, 3, 5):
        assert np.array_equal(step(sl_level(g, g.nodes()[None], p), u), u)


def test_sl_partition_of_unity(P):
    """Weights sum to one (:73-79): a constant state is reproduced."""
    g = P.Grid1D(64)
    c = g.nodes() - np.random.default_rng(1).random(64) * 3 * g.h
    for p in (1, 3, 5):
        assert np.allclose(step(sl_level(g, c[None], p), np.full(64, 2.5)), 2.5, atol=1e-12)


def test_sl_step_constant_shift_exact(P):
    """Integer-cell displacement = pure roll for any p (:104-113)."""
    g = P.Grid1D(32)
    u = np.random.default_rng(1).random(32)
    x = g.nodes()
    for p in (1, 3, 5):
        assert np.allclose(step(sl_level(g, (x - 3 * g.h)[None], p), u), np.roll(u, 3), atol=1e-12)


def test_sl_step_translation_accuracy(P):
    """Fractional constant shift: error decays as h^{p+1} (:116-131)."""
    for p in (1, 3, 5):
        errs, hs = [], []
        for k in (6, 7, 8, 9):
            g = P.Grid1D(2 ** k)
            x = g.nodes()
            u = np.sin(np.pi * x) ** 4
            v = step(sl_level(g, (x - 0.4 * g.h)[None], p), u)
            errs.append(np.max(np.abs(v - np.sin(np.pi * (x - 0.4 * g.h)) ** 4)))
            hs.append(g.h)
        slope = np.polyfit(np.log(hs), np.log(errs), 1)[0]
        assert slope == pytest.approx(p + 1, abs=0.4)


def test_sl_step_2d_separable_shift(P):
    """2D axis-aligned integer shift = 2D roll (:134-145)."""
    g = P.Grid2D(16)
    u = np.random.default_rng(2).random(g.n_points)
    x, y = g.nodes()
    v = step(sl_level(g, ((x - 2 * g.h)[None], (y - 5 * g.h)[None]), 3), u)
    assert np.allclose(v, np.roll(u.reshape(16, 16), (5, 2), axis=(0, 1)).ravel(), atol=1e-12)


def test_sl_step_2d_matches_tensor_of_1d(P):
    """Separable state + axis shifts: 2D step = tensor product of 1D steps (:148-168)."""
    n = 32
    g2, g1 = P.Grid2D(n), P.Grid1D(n)
    xs = g1.nodes()
    ux, uy = np.sin(np.pi * xs) ** 2, np.cos(np.pi * xs) + 2.0
    u = np.outer(uy, ux).ravel()
    x, y = g2.nodes()
    for p in (1, 3, 5):
        v2 = step(sl_level(g2, ((x - 0.3 * g2.h)[None], (y - 0.7 * g2.h)[None]), p), u)
        vx = step(sl_level(g1, (xs - 0.3 * g1.h)[None], p), ux)
        vy = step(sl_level(g1, (xs - 0.7 * g1.h)[None], p), uy)
        assert np.allclose(v2, np.outer(vy, vx).ravel(), atol=1e-12)


def test_sl_rejects_wrong_size(P):
    """State length must match the grid (:186-191)."""
    g = P.Grid1D(32)
    with pytest.raises(ValueError):
        sl_level(g, g.nodes()[None], 1).step(0, torch.zeros(31, dtype=torch.float64).cuda())


# ---- test_coarse_correction.py ----------------------------------------------


def test_apply_ImSD_hand_check_1d(P):
    """(I - diag(1) D_2) e0 = (3, -1, 0, ..., -1) (:98-102), observed through
    the explicit factor 2v - (I - sD)v of a forward-Euler level."""
    g = P.Grid1D(8)
    lv = sl_level(g, g.nodes()[None], 1, kind="forward_euler", sig=np.ones(8))
    v = np.zeros(8)
    v[0] = 1.0
    imsd = 2 * v - step(lv, v)
    assert np.array_equal(imsd, [3.0, -1.0, 0, 0, 0, 0, 0, -1.0])


def test_apply_ImSD_2d_separable(P):
    """With y-coefficients zero the 2D operator is row-wise 1D (:113-127)."""
    g2, g1 = P.Grid2D(8), P.Grid1D(8)
    rng = np.random.default_rng(4)
    v = rng.random(64)
    fx = rng.random(64) * 0.2
    x, y = g2.nodes()
    lv2 = sl_level(g2, (x[None], y[None]), 1, kind="forward_euler", sig=(fx, np.zeros(64)))
    out = 2 * v - step(lv2, v)
    for j in range(8):
        lv1 = sl_level(g1, g1.nodes()[None], 1, kind="forward_euler", sig=fx.reshape(8, 8)[j])
        row = v.reshape(8, 8)[j]
        assert np.allclose(out.reshape(8, 8)[j], 2 * row - step(lv1, row), atol=1e-14)


def test_corrected_step_solves_the_correction_system(P):
    """GMRES(I - diag(s) D) with fixed iterations solves the small-s system
    (cf. test_gmres_solves_spd_system :130-138)."""
    import oracle as O
    g = P.Grid1D(64)
    rng = np.random.default_rng(5)
    for p, scale in ((1, 0.01), (3, 0.05)):
        sig = scale * rng.random(64)
        b = rng.standard_normal(64)
        lv = sl_level(g, g.nodes()[None], p, kind="corrected", sig=sig, gmres=P.GmresConfig(10, None))
        x = step(lv, b)
        # same algorithm as the reference's gmres_solve (oracle restatement)
        xo, _ = O.gmres(lambda v: O.imsd((sig,), O.d_stencil(p), v, 64), b, 10, None)
        assert np.linalg.norm(x - xo) <= 1e-13 * np.linalg.norm(xo)
        if p == 1:   # well conditioned: 10 iterations solve it
            fe = sl_level(g, g.nodes()[None], p, kind="forward_euler", sig=sig)
            Ax = 2 * x - step(fe, x)            # (I - sD) x
            assert np.linalg.norm(Ax - b) <= 1e-10 * np.linalg.norm(b)


def test_corrected_reduces_to_plain_when_sigma_zero(P):
    """sigma = 0 => corrected step = plain SL step (:161-170)."""
    g = P.Grid1D(32)
    c = g.nodes() - 0.5 * g.h
    u = np.sin(np.pi * g.nodes())
    plain = step(sl_level(g, c[None], 1), u)
    corr = step(sl_level(g, c[None], 1, kind="corrected", sig=np.zeros(32), gmres=P.GmresConfig(10, None)), u)
    assert np.allclose(corr, plain, atol=1e-12)


def test_corrected_edge_cases(P):
    """Zero rhs -> zero; non-finite rhs -> ValueError (:150-158)."""
    g = P.Grid1D(16)
    lv = sl_level(g, g.nodes()[None], 1, kind="corrected", sig=np.full(16, 0.1), gmres=P.GmresConfig(10, 1e-2))
    assert np.array_equal(step(lv, np.zeros(16)), np.zeros(16))
    bad = np.ones(16)
    bad[3] = np.nan
    with pytest.raises(ValueError):
        step(lv, bad)
    # the sticky flag was consumed: the level is usable again
    assert np.all(np.isfinite(step(lv, np.ones(16))))


# ---- test_mgrit.py ----------------------------------------------------------


def _base(P, **kw):
    d = dict(n_x=2 ** 5, n_t=2 ** 6, wave_speed="C1", p=1, schedule=4)
    d.update(kw)
    return P.SolverConfig(**d)


def test_hierarchy_level_sizes(P):
    """:16-32"""
    assert [lv.n_steps for lv in P.build_hierarchy(P.SolverConfig(n_x=32, n_t=1024, schedule=4))] == \
        [1024, 256, 64, 16, 4]
    assert [lv.n_steps for lv in P.build_hierarchy(P.SolverConfig(n_x=32, n_t=1024, schedule=4, max_levels=2))] == \
        [1024, 256]
    assert [lv.n_steps for lv in P.build_hierarchy(P.SolverConfig(n_x=32, n_t=2 ** 14, schedule=[16, 4]))] == \
        [16384, 1024, 256, 64, 16, 4]
    with pytest.raises(ValueError):
        P.build_hierarchy(P.SolverConfig(n_x=16, n_t=6, schedule=4))


def test_f_relax_zeroes_f_point_residuals(P):
    """:51-67 (and the exact state is a fixed point)."""
    cfg = _base(P)
    fine = P.build_hierarchy(cfg)[0]
    U = np.random.default_rng(0).random((cfg.n_t + 1, cfg.n_x))
    G = np.zeros_like(U)
    P.f_relax(fine, U, G)
    R = P.residual(fine, U, G)
    fpts = [n for n in range(1, cfg.n_t + 1) if n % fine.cf]
    assert max(np.max(np.abs(R[n])) for n in fpts) <= 1e-12 * np.max(np.abs(U))
    U2 = U.copy()
    P.f_relax(fine, U2, G)
    assert np.array_equal(U, U2)


def test_c_relax_zeroes_c_point_residuals(P):
    """:70-80"""
    cfg = _base(P)
    fine = P.build_hierarchy(cfg)[0]
    U = np.random.default_rng(1).random((cfg.n_t + 1, cfg.n_x))
    G = np.zeros_like(U)
    P.c_relax(fine, U, G)
    R = P.residual(fine, U, G)
    assert max(np.max(np.abs(R[n])) for n in range(fine.cf, cfg.n_t + 1, fine.cf)) <= 1e-12 * np.max(np.abs(U))


def test_f_relax_degenerate_is_sequential(P):
    """m > n_t: one C-interval -> full sequential solve (:83-95)."""
    cfg = _base(P)
    fine = P.build_hierarchy(cfg)[0]
    U = np.zeros((cfg.n_t + 1, cfg.n_x))
    U[0] = P.initial_condition(fine.grid)
    G = np.zeros_like(U)
    P.f_relax(fine, U, G, m=cfg.n_t + 1)
    assert P.space_time_norm(P.residual(fine, U, G)) <= 1e-12


def test_residual_properties(P):
    """Residual KAT and bitwise determinism (:98-112)."""
    cfg = _base(P)
    fine = P.build_hierarchy(cfg)[0]
    U = np.zeros((cfg.n_t + 1, cfg.n_x))
    G = np.zeros_like(U)
    b = np.sin(np.pi * fine.grid.nodes())
    G[1] = b
    R = P.residual(fine, U, G)
    assert np.allclose(R[0], 0.0) and np.allclose(R[1], b) and np.allclose(R[2:], 0.0)
    U = np.random.default_rng(2).random(U.shape)
    assert np.array_equal(P.residual(fine, U, G), P.residual(fine, U, G))


def test_ideal_coarse_operator_one_iteration(P):
    """:115-119"""
    rep, _ = P.solve(_base(P, n_x=2 ** 6, n_t=2 ** 8, max_levels=2, operator_kind="ideal"))
    assert rep.iterations == 1 and rep.status == "converged"


def test_v_cycle_zero_residual_fixed_point(P):
    """:122-132"""
    cfg = _base(P)
    levels = P.build_hierarchy(cfg)
    fine = levels[0]
    U = np.zeros((cfg.n_t + 1, cfg.n_x))
    U[0] = P.initial_condition(fine.grid)
    G = np.zeros_like(U)
    P.f_relax(fine, U, G, m=cfg.n_t + 1)
    U2 = U.copy()
    P.v_cycle(levels, 0, U2, G, "FCF")
    assert P.space_time_norm(U2 - U) <= 1e-10 * P.space_time_norm(U)


def test_solve_matches_sequential_and_is_deterministic(P):
    """:135-149"""
    cfg = _base(P, n_x=2 ** 6, n_t=2 ** 8)
    rep, U = P.solve(cfg)
    assert rep.status == "converged"
    ref = P.sequential_reference(cfg)
    assert P.space_time_norm(U - ref) <= 1e-8 * P.space_time_norm(ref)
    c3 = _base(P, wave_speed="C3")
    r1, u1 = P.solve(c3)
    r2, u2 = P.solve(c3)
    assert np.array_equal(r1.residual_norms, r2.residual_norms) and np.array_equal(u1, u2)
    assert len(r1.residual_norms) == r1.iterations + 1


def test_seed_changes_start_not_answer(P):
    """:152-156"""
    _, u1 = P.solve(_base(P))
    _, u2 = P.solve(_base(P, seed=123))
    assert P.space_time_norm(u1 - u2) <= 1e-7 * P.space_time_norm(u1)


def test_parareal_f_relaxation_differs_from_fcf(P):
    """:159-163"""
    fcf, _ = P.solve(_base(P, max_levels=2))
    f_only, _ = P.solve(_base(P, max_levels=2, relaxation="F"))
    assert f_only.status == "converged" and f_only.residual_norms[1] != fcf.residual_norms[1]


def test_rediscretized_unstable_at_bad_cfl(P):
    """:166-176"""
    g = P.Grid1D(2 ** 6)
    rep, _ = P.solve(P.SolverConfig(n_x=2 ** 6, n_t=2 ** 10, schedule=4, max_levels=2,
                                    operator_kind="rediscretized", departure_policy="erk_rediscretized",
                                    dt=0.7 * g.h))
    assert rep.status == "diverged" or rep.iterations > 50


def test_solve_2d_small(P):
    """:179-184"""
    cfg = P.SolverConfig(n_x=2 ** 4, n_t=2 ** 6, dim=2, wave_speed="C5", p=1, schedule=4)
    rep, U = P.solve(cfg)
    assert rep.status == "converged"
    ref = P.sequential_reference(cfg)
    assert P.space_time_norm(U - ref) <= 1e-8 * P.space_time_norm(ref)


def test_constant_speed_shares_departures(P):
    """:187-192"""
    lv = P.build_hierarchy(_base(P))[0]
    assert lv.shared and lv.s_x.shape[0] == 1
    lv = P.build_hierarchy(_base(P, wave_speed="C2"))[0]
    assert not lv.shared and lv.s_x.shape[0] == 2 ** 6
