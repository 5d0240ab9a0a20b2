"""Where does a solve's time go besides the V-cycle kernels?  For one bench
config: the device-loop solve (one graph launch per solve), the eager
host-driven loop (use_graph=False: launches + a host sync per iteration), and
the solve's prologue pieces.  Usage: python tools/overhead_probe.py [cfg2]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2203_13382_b200 as P  # noqa: E402
from paper_2203_13382_b200 import mgrit as M  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
cfg = P.SolverConfig(**bench.CONFIGS[name])
levels = P.build_hierarchy(cfg)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def timed(fn, reps=5):
    best = None
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e0.record()
        out = fn()
        e1.record()
        torch.cuda.synchronize()
        t = (e0.elapsed_time(e1), (time.perf_counter() - t0) * 1e3, out)
        best = t if best is None or t[0] < best[0] else best
    return best


for g in (True, False):
    for _ in range(2):
        P.solve(cfg, levels, output="device", use_graph=g)
dev_ms, wall_ms, rep = timed(lambda: P.solve(cfg, levels, output="device", use_graph=True)[0])
k = rep.iterations
print(f"{name}: iterations {k} ({rep.status}); device-loop solve {dev_ms:.3f} ms (wall {wall_ms:.3f})")
dev2, wall2, rep2 = timed(lambda: P.solve(cfg, levels, output="device", use_graph=False)[0])
assert rep2.iterations == k and list(rep2.residual_norms) == list(rep.residual_norms)
print(f"  eager host loop {dev2:.3f} ms: {(dev2 - dev_ms) / k * 1e3:.1f} us/iteration more; histories identical")

sess = next(iter(levels[0].__dict__["_sessions"].values()))
grid = levels[0].grid
fine = levels[0]
row_ss = sess.row_ss
parts = {
    "U[0] = u0 (cached row)": lambda: sess.U[0].copy_(M._initial_row(cfg, fine, sess.U.device)),
    "pcg64 fill": lambda: M.pcg64_uniform(cfg.seed, cfg.n_t, grid.n_points, sess.U[1:], pm1=(cfg.iterate == "pm1")),
    "r0 rows + sum": lambda: (fine._apply(sess.U, 0, 1, cfg.n_t, None, U_sub=sess.U[1:], row_sumsq=row_ss),
                              M.device_sum(row_ss)),
    "U.clone": lambda: sess.U.clone(),
}
for key, fn in parts.items():
    d, w, _ = timed(fn)
    print(f"  {key}: device {d:.3f} ms, wall {w:.3f} ms")
