"""Generate golden fixtures by running the REAL reference (mgrit_advect).

Run in the build container only (the reference is not on the GPU box):

    NUMBA_CACHE_DIR=/tmp/numba PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_golden.py [ops] [solves] [accept] [big]

The reference is imported from a scratch copy (baseline/_ref/src, git-ignored)
or, failing that, /root/reference/pkg/src.  Outputs are small .npz files in this
directory plus index.json; the CPU test-suite pins the oracle against them and
the GPU test-suite pins the CUDA path against them.

BASELINE configs use the reference's public WaveSpeed closure API for the
non-catalog speeds and a twin of ``mgrit.solve`` (same v_cycle / residual /
norm calls) that accepts BASELINE's initial state and initial iterate
(SURVEY.md Appendix A).
"""

from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
for cand in (os.path.join(REPO, "baseline", "_ref", "src"), "/root/reference/pkg/src"):
    if os.path.isdir(os.path.join(cand, "mgrit_advect")):
        sys.path.insert(0, cand)
        break
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.dont_write_bytecode = True

import mgrit_advect as R  # noqa: E402
from mgrit_advect import mgrit as RM  # noqa: E402

TWO_PI = 2.0 * np.pi
SPEEDS = {
    "B2": R.WaveSpeed("B2", 1, (lambda x, t: 1.0 + 0.5 * np.sin(TWO_PI * x) * np.cos(TWO_PI * t),)),
    "B4": R.WaveSpeed("B4", 2, (
        lambda x, y, t: np.cos(np.pi * x) ** 2 * np.cos(TWO_PI * t) + 0.5,
        lambda x, y, t: np.sin(np.pi * y) ** 2 * np.cos(TWO_PI * t) + 0.5,
    )),
}


def _speed(name):
    return SPEEDS.get(name, name)


def ref_cfg(kw):
    kw = dict(kw)
    kw.pop("u0", None)
    kw.pop("iterate", None)
    kw["wave_speed"] = _speed(kw.get("wave_speed", "C1"))
    return RM.SolverConfig(**kw)


def ref_u0(cfg, u0):
    grid = R.Grid1D(cfg.n_x) if cfg.dim == 1 else R.Grid2D(cfg.n_x)
    if cfg.dim == 2 and u0 == "sin4":
        x, y = grid.nodes()
        return np.sin(np.pi * x) ** 4 * np.sin(np.pi * y) ** 4
    return R.initial_condition(grid)


def ref_solve(kw, snapshots=False, count_gmres=False):
    """Twin of mgrit.solve (mgrit.py:337-378) with BASELINE u0/iterate hooks."""
    cfg = ref_cfg(kw)
    t0 = time.perf_counter()
    levels = RM.build_hierarchy(cfg)
    t_build = time.perf_counter() - t0
    counts = []
    orig = RM.gmres_solve
    if count_gmres:
        def wrapped(op, rhs, gcfg):
            x, hist = orig(op, rhs, gcfg)
            counts.append(len(hist) - 1)
            return x, hist
        RM.gmres_solve = wrapped
    try:
        fine = levels[0]
        U = np.empty((cfg.n_t + 1, fine.grid.n_points))
        U[0] = ref_u0(cfg, kw.get("u0", "reference"))
        X = np.random.default_rng(cfg.seed).random((cfg.n_t, fine.grid.n_points))
        if kw.get("iterate", "uniform01") == "pm1":
            X = 2.0 * X - 1.0
        U[1:] = X
        G = np.zeros_like(U)
        t1 = time.perf_counter()
        r0 = R.space_time_norm(RM.residual(fine, U, G))
        hist = [r0]
        snaps = []
        status = "max_iters"
        for _ in range(cfg.max_iters):
            try:
                RM.v_cycle(levels, 0, U, G, cfg.relaxation)
                r = R.space_time_norm(RM.residual(fine, U, G))
            except (ValueError, FloatingPointError):
                hist.append(float("nan"))
                status = "diverged"
                break
            hist.append(r)
            if snapshots:
                snaps.append(U.copy())
            if not np.isfinite(r) or r >= cfg.divergence_factor * r0:
                status = "diverged"
                break
            if r <= cfg.rtol * r0:
                status = "converged"
                break
        t_solve = time.perf_counter() - t1
    finally:
        RM.gmres_solve = orig
    return dict(levels=levels, U=U, hist=np.array(hist), status=status, snaps=snaps,
                counts=counts, t_build=t_build, t_solve=t_solve,
                sizes=[lv.n_steps for lv in levels])


INDEX_PATH = os.path.join(HERE, "index.json")


def _load_index():
    if os.path.exists(INDEX_PATH):
        with open(INDEX_PATH) as f:
            return json.load(f)
    return {}


def _save_index(ix):
    with open(INDEX_PATH, "w") as f:
        json.dump(ix, f, indent=1, sort_keys=True)


def record_solve(name, kw, row_stride=None, snapshots=False, count_gmres=False, note=""):
    print(f"[golden] solve {name} {kw}", flush=True)
    out = ref_solve(kw, snapshots=snapshots, count_gmres=count_gmres)
    U = out["U"]
    arrays = dict(hist=out["hist"], row_norms=np.linalg.norm(U, axis=1))
    if row_stride is None:
        arrays["U"] = U
    else:
        arrays["U_rows"] = U[::row_stride]
    if snapshots:
        arrays["snaps"] = np.stack(out["snaps"])
    if count_gmres:
        arrays["gmres_counts"] = np.array(out["counts"], dtype=np.int32)
    np.savez_compressed(os.path.join(HERE, f"solve_{name}.npz"), **arrays)
    ix = _load_index()
    ix[name] = dict(kw=kw, iterations=len(out["hist"]) - 1, status=out["status"],
                    row_stride=row_stride, levels=out["sizes"], note=note,
                    ref_build_s=round(out["t_build"], 3), ref_solve_s=round(out["t_solve"], 3))
    _save_index(ix)
    print(f"  -> {ix[name]['iterations']} it, {out['status']}, solve {out['t_solve']:.1f}s", flush=True)


# ---------------------------------------------------------------------------


def make_ops():
    """Per-operator vectors on seeded inputs (1D and 2D, p = 1, 3, 5)."""
    rng = np.random.default_rng(20220325)
    arrays = {}
    # decompose + weights on adversarial coordinates (nodes, near-nodes, wraps)
    for n in (16, 64, 1024):
        g = R.Grid1D(n)
        base = g.nodes()
        c = np.concatenate([
            rng.uniform(-5, 5, 4000),
            base, base + 1e-17, base - 1e-17, base + g.h * 0.5,
            np.array([-1.0, 1.0, 3.0, -3.0, 1.0 - 1e-16, -1.0 + 1e-16, 0.0, -0.0]),
        ])
        e, eps = R.decompose(g, c)
        arrays[f"dec_n{n}_coords"] = c
        arrays[f"dec_n{n}_east"] = e
        arrays[f"dec_n{n}_eps"] = eps
    for p in (1, 3, 5):
        eps = np.concatenate([rng.random(3000), [0.0, 0.5, 1 - 1e-16, 1e-300]])
        arrays[f"w_p{p}_eps"] = eps
        arrays[f"w_p{p}"] = R.interp_weights(p, eps)
    # ERK departures (1D: C1, C2, C3, B2 ; 2D: C4, C5, B4) and SL steps
    for speed, dim, n in (("C1", 1, 64), ("C2", 1, 64), ("C3", 1, 64), ("B2", 1, 128),
                          ("C4", 2, 16), ("C5", 2, 16), ("B4", 2, 24)):
        ws = _speed(speed) if speed in SPEEDS else R.get_wave_speed(speed)
        grid = R.Grid1D(n) if dim == 1 else R.Grid2D(n)
        for order in (1, 3, 5):
            dt = 0.85 * grid.h * (1.0 + 3.0 * (order == 5))
            t0 = 0.37
            dep = R.erk_departures(grid, ws, t0, dt, R.erk_scheme(order))
            key = f"erk_{speed}_r{order}"
            if dim == 1:
                arrays[key + "_east"] = dep.east
                arrays[key + "_eps"] = dep.eps
                arrays[key + "_disp"] = dep.displacement
            else:
                arrays[key + "_east"] = np.stack([dep.east_x, dep.east_y])
                arrays[key + "_eps"] = np.stack([dep.eps, dep.nu])
                arrays[key + "_disp"] = np.stack([dep.displacement_x, dep.displacement_y])
            u = rng.standard_normal(grid.n_points)
            arrays[key + "_u"] = u
            for p in (1, 3, 5):
                arrays[key + f"_sl_p{p}"] = R.sl_step(grid, dep, p, u)
    # GMRES on I - diag(sigma) D (1D and 2D), fixed and tolerance modes
    for dim, n in ((1, 64), (1, 256), (2, 16)):
        grid = R.Grid1D(n) if dim == 1 else R.Grid2D(n)
        for p in (1, 3, 5):
            for scale in (0.0, 0.05, 0.6):
                sx = scale * rng.standard_normal(grid.n_points)
                field = R.CorrectionField(sx) if dim == 1 else R.CorrectionField(
                    sx, scale * rng.standard_normal(grid.n_points))
                st = R.derivative_stencil(p)
                rhs = rng.standard_normal(grid.n_points)
                key = f"gm_d{dim}_n{n}_p{p}_s{scale}"
                arrays[key + "_sx"] = field.x
                if dim == 2:
                    arrays[key + "_sy"] = field.y
                arrays[key + "_rhs"] = rhs
                arrays[key + "_imsd"] = R.coarse_correction.apply_ImSD(field, st, rhs, grid)
                for mode, cfgm in (("fixed", R.GmresConfig(10, None)), ("tol", R.GmresConfig(10, 1e-2))):
                    x, hist = R.gmres_solve(lambda v: R.coarse_correction.apply_ImSD(field, st, v, grid), rhs, cfgm)
                    arrays[key + f"_{mode}_x"] = x
                    arrays[key + f"_{mode}_hist"] = hist
    np.savez_compressed(os.path.join(HERE, "ops.npz"), **arrays)
    print(f"[golden] ops.npz: {len(arrays)} arrays", flush=True)


def make_hierarchies():
    """Departure records + sigma of small hierarchies (backtracking, phi/sigma)."""
    arrays = {}
    cases = {
        "h1_C3_p3_m4": dict(n_x=32, n_t=64, wave_speed="C3", p=3, schedule=4),
        "h1_B2_p5_m8": dict(n_x=64, n_t=128, wave_speed="B2", p=5, schedule=8),
        "h1_C1_p1_m8": dict(n_x=64, n_t=256, wave_speed="C1", p=1, schedule=8, max_levels=2),
        "h2_C5_p3_m4": dict(n_x=16, n_t=64, dim=2, wave_speed="C5", p=3, schedule=4),
        "h2_B4_p5_m8": dict(n_x=16, n_t=128, dim=2, wave_speed="B4", p=5, schedule=8),
    }
    meta = {}
    for name, kw in cases.items():
        levels = RM.build_hierarchy(ref_cfg(kw))
        meta[name] = dict(kw=kw, sizes=[lv.n_steps for lv in levels])
        for li, lv in enumerate(levels):
            if lv.departures is None:
                continue
            if lv.grid.dim == 1:
                arrays[f"{name}_L{li}_east"] = np.stack([d.east for d in lv.departures])
                arrays[f"{name}_L{li}_eps"] = np.stack([d.eps for d in lv.departures])
                arrays[f"{name}_L{li}_disp"] = np.stack([d.displacement for d in lv.departures])
            else:
                arrays[f"{name}_L{li}_east"] = np.stack([np.stack([d.east_x, d.east_y]) for d in lv.departures])
                arrays[f"{name}_L{li}_eps"] = np.stack([np.stack([d.eps, d.nu]) for d in lv.departures])
                arrays[f"{name}_L{li}_disp"] = np.stack(
                    [np.stack([d.displacement_x, d.displacement_y]) for d in lv.departures])
            if lv.sigma is not None:
                if lv.grid.dim == 1:
                    arrays[f"{name}_L{li}_sigma"] = np.stack([s.x for s in lv.sigma])
                else:
                    arrays[f"{name}_L{li}_sigma"] = np.stack([np.stack([s.x, s.y]) for s in lv.sigma])
    np.savez_compressed(os.path.join(HERE, "hier.npz"), **arrays)
    with open(os.path.join(HERE, "hier.json"), "w") as f:
        json.dump(meta, f, indent=1, sort_keys=True)
    print(f"[golden] hier.npz: {len(arrays)} arrays", flush=True)


SMALL_SOLVES = {
    # tiny cases with per-iteration snapshots (rel-1e-12 iterate parity per iteration)
    "tiny1d_C3_p3_m4": (dict(n_x=32, n_t=64, wave_speed="C3", p=3, schedule=4), dict(snapshots=True, count_gmres=True)),
    "tiny1d_B2_p5_m8": (dict(n_x=64, n_t=128, wave_speed="B2", p=5, schedule=8, seed=2), dict(snapshots=True, count_gmres=True)),
    "tiny1d_C1_2lvl_pm1": (dict(n_x=64, n_t=256, wave_speed="C1", p=1, schedule=8, max_levels=2, iterate="pm1"), dict(snapshots=True)),
    "tiny2d_C5_p3_m4": (dict(n_x=16, n_t=64, dim=2, wave_speed="C5", p=3, schedule=4), dict(snapshots=True, count_gmres=True)),
    "tiny2d_B4_p3_m4": (dict(n_x=16, n_t=64, dim=2, wave_speed="B4", p=3, schedule=4, u0="sin4", seed=3), dict(snapshots=True, count_gmres=True)),
    # operator kinds / policies / relaxation variants
    "kind_F_relax": (dict(n_x=32, n_t=64, wave_speed="C2", p=1, schedule=4, relaxation="F"), {}),
    "kind_ideal": (dict(n_x=64, n_t=256, wave_speed="C1", p=1, schedule=4, max_levels=2, operator_kind="ideal"), {}),
    "kind_rediscretized": (dict(n_x=64, n_t=256, wave_speed="C3", p=3, schedule=4, operator_kind="rediscretized",
                                departure_policy="erk_rediscretized", max_iters=30), {}),
    "kind_forward_euler": (dict(n_x=64, n_t=256, wave_speed="C1", p=1, schedule=4, max_levels=2,
                                operator_kind="forward_euler", max_iters=30), {}),
    "kind_erk_substeps": (dict(n_x=32, n_t=128, wave_speed="C3", p=3, schedule=4, departure_policy="erk_substeps"), {}),
    "kind_schedule_16_4": (dict(n_x=32, n_t=1024, wave_speed="C3", p=1, schedule=[16, 4]), dict(count_gmres=True)),
    "kind_diverge": (dict(n_x=64, n_t=1024, schedule=4, max_levels=2, operator_kind="rediscretized",
                          departure_policy="erk_rediscretized", dt=0.7 * 2.0 / 64), {}),
    # BASELINE configs at reduced size (same p, m, speed, seed, dt/h, u0, iterate)
    "cfg3_reduced": (dict(n_x=1024, n_t=1024, wave_speed="B2", p=5, schedule=8, seed=2), dict(count_gmres=True)),
    "cfg4_reduced": (dict(n_x=32, n_t=256, dim=2, wave_speed="B4", p=3, schedule=4, seed=3, u0="sin4"), dict(count_gmres=True)),
    "cfg5_reduced": (dict(n_x=32, n_t=512, dim=2, wave_speed="B4", p=5, schedule=8, seed=4, u0="sin4"), dict(count_gmres=True)),
}

ACCEPT = {}
for _s, _p, _m in [("C1", 1, 4), ("C1", 1, 8), ("C1", 1, 16), ("C1", 3, 4), ("C1", 5, 4), ("C2", 1, 4), ("C3", 1, 4), ("C3", 5, 16)]:
    ACCEPT[f"crit1_{_s}_p{_p}_m{_m}"] = dict(n_x=2**8, n_t=2**10, wave_speed=_s, p=_p, schedule=_m, max_levels=2)
for _s, _p, _m in [("C1", 1, 4), ("C1", 3, 4), ("C1", 5, 4), ("C3", 5, 16)]:
    ACCEPT[f"crit2_{_s}_p{_p}_m{_m}"] = dict(n_x=2**8, n_t=2**10, wave_speed=_s, p=_p, schedule=_m)
for _s, _p, _m in [("C4", 1, 4), ("C4", 3, 4), ("C4", 5, 16), ("C5", 1, 4)]:
    ACCEPT[f"crit3_{_s}_p{_p}_m{_m}"] = dict(n_x=2**6, n_t=2**10, dim=2, wave_speed=_s, p=_p, schedule=_m)

BIG = {
    "cfg1_full": (dict(n_x=1024, n_t=1024, wave_speed="C1", p=1, schedule=8, max_levels=2, dt=2.0 / 1024, seed=0,
                       iterate="pm1"), 8, "BASELINE config 1 as written (CFL 1, degenerate)"),
    "cfg1_085h": (dict(n_x=1024, n_t=1024, wave_speed="C1", p=1, schedule=8, max_levels=2, seed=0, iterate="pm1"), 8,
                  "BASELINE config 1 mesh at the reference default dt = 0.85h (non-degenerate companion)"),
    "cfg2_full": (dict(n_x=4096, n_t=4096, wave_speed="B2", p=3, schedule=4, seed=1), 64,
                  "BASELINE config 2 at full size, dt = 0.85h (reference default)"),
}


def main(argv):
    what = set(argv) or {"ops", "solves"}
    if "ops" in what:
        make_ops()
        make_hierarchies()
    if "solves" in what:
        for name, (kw, opts) in SMALL_SOLVES.items():
            record_solve(name, kw, **opts)
    if "accept" in what:
        for name, kw in ACCEPT.items():
            record_solve(name, kw, row_stride=32, note="reference acceptance-suite cell (test_acceptance.py)")
    if "big" in what:
        for name, (kw, stride, note) in BIG.items():
            record_solve(name, kw, row_stride=stride, note=note)


if __name__ == "__main__":
    main(sys.argv[1:])
