"""Pin the CPU oracle against vectors produced by the real reference
(tests/golden/make_golden.py).  CPU only."""

import numpy as np
import pytest

import oracle as O
from conftest import load_solve


def test_decompose_matches_reference(ops):
    for n in (16, 64, 1024):
        e, eps = O.decompose(n, ops[f"dec_n{n}_coords"])
        assert np.array_equal(e, ops[f"dec_n{n}_east"])
        assert np.array_equal(eps, ops[f"dec_n{n}_eps"])


@pytest.mark.parametrize("p", [1, 3, 5])
def test_weights_match_reference(ops, p):
    assert np.array_equal(O.lagrange_weights(p, ops[f"w_p{p}_eps"]), ops[f"w_p{p}"])


SPEEDS = (("C1", 1, 64), ("C2", 1, 64), ("C3", 1, 64), ("B2", 1, 128), ("C4", 2, 16), ("C5", 2, 16), ("B4", 2, 24))


@pytest.mark.parametrize("speed,dim,n", SPEEDS)
@pytest.mark.parametrize("order", [1, 3, 5])
def test_erk_and_sl_match_reference(ops, speed, dim, n, order):
    h = 2.0 / n
    dt = 0.85 * h * (1.0 + 3.0 * (order == 5))
    dep = O.erk_departures(dim, n, speed, 0.37, dt, order)
    key = f"erk_{speed}_r{order}"
    east = np.stack(dep.east) if dim == 2 else dep.east[0]
    eps = np.stack(dep.eps) if dim == 2 else dep.eps[0]
    disp = np.stack(dep.disp) if dim == 2 else dep.disp[0]
    assert np.array_equal(east, ops[key + "_east"])
    assert np.array_equal(eps, ops[key + "_eps"])
    assert np.array_equal(disp, ops[key + "_disp"])
    for p in (1, 3, 5):
        out = O.sl_apply(dim, n, p, dep, ops[key + "_u"])
        assert np.array_equal(out, ops[key + f"_sl_p{p}"]), (key, p)


def _gmres_cases(ops):
    for dim, n in ((1, 64), (1, 256), (2, 16)):
        for p in (1, 3, 5):
            for scale in (0.0, 0.05, 0.6):
                yield dim, n, p, scale


def test_imsd_and_gmres_match_reference(ops):
    for dim, n, p, scale in _gmres_cases(ops):
        key = f"gm_d{dim}_n{n}_p{p}_s{scale}"
        sig = (ops[key + "_sx"],) if dim == 1 else (ops[key + "_sx"], ops[key + "_sy"])
        c = O.d_stencil(p)
        rhs = ops[key + "_rhs"]
        assert np.array_equal(O.imsd(sig, c, rhs, n), ops[key + "_imsd"]), key
        for mode, tol in (("fixed", None), ("tol", 1e-2)):
            x, hist = O.gmres(lambda v: O.imsd(sig, c, v, n), rhs, 10, tol)
            assert np.array_equal(x, ops[key + f"_{mode}_x"]), (key, mode)
            assert np.array_equal(hist, ops[key + f"_{mode}_hist"]), (key, mode)


def test_hierarchies_match_reference(hier):
    meta, arr = hier
    for name, info in meta.items():
        cfg = O.OConfig(**info["kw"])
        levels = O.hierarchy(cfg)
        assert [lv.n_steps for lv in levels] == info["sizes"]
        for li, lv in enumerate(levels):
            if lv.deps is None:
                continue
            pick = (lambda d, f: f(d)[0]) if lv.dim == 1 else (lambda d, f: np.stack(f(d)))
            assert np.array_equal(np.stack([pick(d, lambda d: d.east) for d in lv.deps]), arr[f"{name}_L{li}_east"])
            assert np.array_equal(np.stack([pick(d, lambda d: d.eps) for d in lv.deps]), arr[f"{name}_L{li}_eps"])
            assert np.array_equal(np.stack([pick(d, lambda d: d.disp) for d in lv.deps]), arr[f"{name}_L{li}_disp"])
            if lv.sigma is not None:
                sig = np.stack([s[0] if lv.dim == 1 else np.stack(s) for s in lv.sigma])
                assert np.array_equal(sig, arr[f"{name}_L{li}_sigma"]), (name, li)


FAST_SOLVES = ["tiny1d_C3_p3_m4", "tiny1d_B2_p5_m8", "tiny1d_C1_2lvl_pm1", "kind_F_relax", "kind_ideal",
               "kind_rediscretized", "kind_forward_euler", "kind_erk_substeps", "tiny2d_C5_p3_m4",
               "crit1_C1_p1_m8", "crit1_C3_p5_m16", "crit2_C1_p3_m4", "cfg1_full", "cfg1_085h"]


@pytest.mark.parametrize("name", FAST_SOLVES)
def test_oracle_solve_matches_reference(golden_index, name):
    """The oracle reproduces the reference's residual history and iterate
    bit-for-bit (same numpy/BLAS calls; C sweep == numba sweep)."""
    info = golden_index[name]
    g = load_solve(name)
    rep, U = O.solve(O.OConfig(**info["kw"]))
    assert rep.iterations == info["iterations"]
    assert rep.status == info["status"]
    assert np.array_equal(rep.residual_norms, g["hist"])
    if "U" in g:
        assert np.array_equal(U, g["U"])
    else:
        assert np.array_equal(U[:: info["row_stride"]], g["U_rows"])


def test_oracle_snapshots_match_reference():
    g = load_solve("tiny1d_C3_p3_m4")
    snaps = []
    O.solve(O.OConfig(n_x=32, n_t=64, wave_speed="C3", p=3, schedule=4), on_iter=lambda k, U: snaps.append(U.copy()))
    assert np.array_equal(np.stack(snaps), g["snaps"])


def test_oracle_gmres_counts_match_reference():
    g = load_solve("tiny1d_C3_p3_m4")
    rep, _ = O.solve(O.OConfig(n_x=32, n_t=64, wave_speed="C3", p=3, schedule=4), log_gmres=True)
    assert rep.gmres_counts == list(g["gmres_counts"])


def test_reference_acceptance_counts_recorded(golden_index):
    """The reference's own recorded counts (pkg/test_output.txt:124-130) are
    what the golden generator reproduced."""
    expect = {"crit1_C1_p1_m4": 12, "crit1_C1_p1_m8": 10, "crit1_C1_p1_m16": 9, "crit1_C1_p3_m4": 20,
              "crit1_C1_p5_m4": 28, "crit1_C2_p1_m4": 10, "crit1_C3_p1_m4": 10, "crit1_C3_p5_m16": 15,
              "crit2_C1_p1_m4": 13, "crit2_C1_p3_m4": 21, "crit2_C1_p5_m4": 30, "crit2_C3_p5_m16": 15,
              "crit3_C4_p1_m4": 12, "crit3_C4_p3_m4": 20, "crit3_C4_p5_m16": 16, "crit3_C5_p1_m4": 10}
    for k, v in expect.items():
        assert golden_index[k]["iterations"] == v, k
