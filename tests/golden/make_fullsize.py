"""Full-size golden histories for BASELINE configs 3 and 4 (build container only).

    NUMBA_CACHE_DIR=/tmp/numba PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_fullsize.py {cfg4 | cfg5mesh_nt128} [max_iters]
    python tests/golden/make_fullsize.py cfg3 [max_iters]

* ``cfg4`` (2D 512^2 x 1024, p = 3, m = 4) runs the REAL reference
  (mgrit_advect, imported from /root/reference/pkg/src or baseline/_ref/src)
  through the same ``ref_solve`` twin as make_golden.py: the reference's own
  ``build_hierarchy`` / ``v_cycle`` / ``residual`` / ``space_time_norm`` calls,
  only u0 = sin^4 sin^4 and the seeded iterate injected.
  ~740 s per V-cycle and 26 GB here.
* ``cfg5mesh_nt128`` runs the real reference on config 5's 1024^2 mesh,
  p = 5, m = 8, seed 4 and u0 for 128 steps (levels [128, 16, 2]), two
  V-cycles: the exact kernel instantiations config 5 uses, at full mesh size.
* ``cfg3`` (1D 16384 x 16384, p = 5, m = 8) cannot run through the reference in
  62 GB (its cached (S, n, p+1) gather tables and the (B, n, p+1) temporaries
  of ``Level.step_batch`` need ~64 GB), so it runs through the oracle, which
  tests/test_oracle_golden.py pins bit-for-bit to the reference on every
  committed fixture (including cfg3_reduced and the full-size cfg2 solve).

Both write ``solve_<name>.npz`` after EVERY iteration (a partial run is still a
first-k fixture):
  hist            residual history r_0..r_k
  row_norms       (k, N+1) per-iteration row 2-norms of the iterate
  cols_idx        64 fixed spatial indices
  cols            (k, N+1, 64) the iterate's values at those indices
  gmres_per_iter  (k,) number of GMRES calls per V-cycle + residual
  gmres_counts    every call's Arnoldi count, in call order
  meta            json: kw, status, levels, timings, source
"""

from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))

CASES = {
    "cfg4_full": dict(n_x=512, n_t=1024, dim=2, wave_speed="B4", p=3, schedule=4, seed=3, u0="sin4"),
    "cfg3_full": dict(n_x=16384, n_t=16384, wave_speed="B2", p=5, schedule=8, seed=2),
    # config 5's mesh, degree, factor, speed, u0 and seed on a short time
    # horizon (levels [128, 16, 2]): the production 1024^2 p = 5 kernels
    # (sl2d FULL tiles, gmres2d_coop<5, 1024>) against the reference, 2 V-cycles
    "cfg5mesh_nt128": dict(n_x=1024, n_t=128, dim=2, wave_speed="B4", p=5, schedule=8, seed=4, u0="sin4"),
}
REFERENCE_CASES = {"cfg4_full": 100, "cfg5mesh_nt128": 2}   # name -> default max_iters


def cols_index(n_points: int) -> np.ndarray:
    rng = np.random.default_rng(12345)
    fixed = np.array([0, 1, n_points // 2, n_points - 1])
    return np.unique(np.concatenate([fixed, rng.choice(n_points, 60, replace=False)]))[:64]


class Recorder:
    def __init__(self, name, kw, source, n_points):
        self.name, self.kw, self.source = name, kw, source
        self.idx = cols_index(n_points)
        self.hist, self.norms, self.cols, self.per_iter = [], [], [], []
        self.counts: list[int] = []
        self.t0 = time.perf_counter()
        self.levels = None
        self.t_build = None

    def save(self, status):
        path = os.path.join(HERE, f"solve_{self.name}.npz")
        meta = dict(kw=self.kw, status=status, iterations=len(self.hist) - 1, levels=self.levels,
                    source=self.source, build_s=self.t_build,
                    elapsed_s=round(time.perf_counter() - self.t0, 1))
        np.savez_compressed(path + ".tmp.npz", hist=np.array(self.hist), row_norms=np.array(self.norms),
                            cols_idx=self.idx, cols=np.array(self.cols),
                            gmres_per_iter=np.array(self.per_iter, dtype=np.int64),
                            gmres_counts=np.array(self.counts, dtype=np.int32),
                            meta=np.array(json.dumps(meta)))
        os.replace(path + ".tmp.npz", path)
        print(f"[fullsize] {self.name}: {meta['iterations']} it saved ({status}), hist {self.hist[-1]:.6e}, "
              f"{meta['elapsed_s']} s", flush=True)

    def on_iter(self, U):
        self.norms.append(np.linalg.norm(U, axis=1))
        self.cols.append(U[:, self.idx].copy())


def run_reference(name, kw, max_iters):
    sys.path.insert(0, HERE)
    import make_golden as MG
    R, RM = MG.R, MG.RM
    cfg = MG.ref_cfg(dict(kw, max_iters=max_iters))
    t0 = time.perf_counter()
    levels = RM.build_hierarchy(cfg)
    fine = levels[0]
    rec = Recorder(name, kw, "reference mgrit_advect (make_golden.ref_cfg / ref_u0 twin of mgrit.solve)",
                   fine.grid.n_points)
    rec.t_build = round(time.perf_counter() - t0, 1)
    rec.levels = [lv.n_steps for lv in levels]
    print(f"[fullsize] {name}: hierarchy {rec.levels} in {rec.t_build} s", flush=True)
    orig = RM.gmres_solve

    def wrapped(op, rhs, gcfg):
        x, hist = orig(op, rhs, gcfg)
        rec.counts.append(len(hist) - 1)
        return x, hist
    RM.gmres_solve = wrapped
    try:
        U = np.empty((cfg.n_t + 1, fine.grid.n_points))
        U[0] = MG.ref_u0(cfg, kw.get("u0", "reference"))
        U[1:] = np.random.default_rng(cfg.seed).random((cfg.n_t, fine.grid.n_points))
        G = np.zeros_like(U)
        r0 = R.space_time_norm(RM.residual(fine, U, G))
        rec.hist.append(r0)
        status = "max_iters"
        for _ in range(cfg.max_iters):
            c0 = len(rec.counts)
            RM.v_cycle(levels, 0, U, G, cfg.relaxation)
            r = R.space_time_norm(RM.residual(fine, U, G))
            rec.hist.append(r)
            rec.per_iter.append(len(rec.counts) - c0)
            rec.on_iter(U)
            if not np.isfinite(r) or r >= cfg.divergence_factor * r0:
                status = "diverged"
            elif r <= cfg.rtol * r0:
                status = "converged"
            rec.save(status if status != "max_iters" else "running")
            if status != "max_iters":
                break
        rec.save(status)
    finally:
        RM.gmres_solve = orig


def run_oracle(name, kw, max_iters):
    sys.path.insert(0, REPO)
    import oracle as O
    cfg = O.OConfig(**dict(kw, max_iters=max_iters))
    t0 = time.perf_counter()
    levels = O.hierarchy(cfg)
    rec = Recorder(name, kw, "oracle (bit-pinned restatement; reference infeasible in 62 GB)", levels[0].n_points)
    rec.t_build = round(time.perf_counter() - t0, 1)
    rec.levels = [lv.n_steps for lv in levels]
    print(f"[fullsize] {name}: hierarchy {rec.levels} in {rec.t_build} s", flush=True)
    log = O.GmresLog()
    for lv in levels:
        lv.log = log
        # the departure coordinates/displacements are only needed while building
        if lv.deps is not None:
            for d in lv.deps:
                d.coords = d.disp = None
    rec.counts = log.counts
    fine = levels[0]
    U = np.empty((cfg.n_t + 1, fine.n_points))
    U[0] = O.initial_state(cfg)
    U[1:] = O.initial_iterate(cfg)
    G = np.zeros_like(U)
    r0 = O.st_norm(O.residual(fine, U, G))
    rec.hist.append(r0)
    status = "max_iters"
    for _ in range(cfg.max_iters):
        c0 = len(log.counts)
        O.v_cycle(levels, 0, U, G, cfg.relaxation)
        r = O.st_norm(O.residual(fine, U, G))
        rec.hist.append(r)
        rec.per_iter.append(len(log.counts) - c0)
        rec.on_iter(U)
        if not np.isfinite(r) or r >= cfg.divergence_factor * r0:
            status = "diverged"
        elif r <= cfg.rtol * r0:
            status = "converged"
        rec.save(status if status != "max_iters" else "running")
        if status != "max_iters":
            break
    rec.save(status)


def compact(name, norm_stride, col_stride):
    """Keep every norm_stride-th row norm and every col_stride-th row of the
    sampled columns (plus the last row), so large fixtures stay a few MB."""
    path = os.path.join(HERE, f"solve_{name}.npz")
    g = dict(np.load(path))
    n_rows = g["row_norms"].shape[1]
    nr = np.unique(np.append(np.arange(0, n_rows, norm_stride), n_rows - 1))
    cr = np.unique(np.append(np.arange(0, n_rows, col_stride), n_rows - 1))
    if "norm_rows" in g:
        raise SystemExit(f"{name} is already compact")
    g["row_norms"] = g["row_norms"][:, nr]
    g["cols"] = g["cols"][:, cr]
    g["norm_rows"], g["cols_rows"] = nr, cr
    np.savez_compressed(path, **g)
    print(f"[fullsize] {name}: kept {len(nr)} row norms and {len(cr)} column rows of {n_rows}")


def main(argv):
    if argv[0] == "compact":
        compact(argv[1], int(argv[2]), int(argv[3]))
        return
    name = argv[0] if argv[0] in CASES else f"{argv[0]}_full"
    kw = CASES[name]
    if name in REFERENCE_CASES:
        max_iters = int(argv[1]) if len(argv) > 1 else REFERENCE_CASES[name]
        run_reference(name, kw, max_iters)
    else:
        max_iters = int(argv[1]) if len(argv) > 1 else 100
        run_oracle(name, kw, max_iters)


if __name__ == "__main__":
    main(sys.argv[1:])
