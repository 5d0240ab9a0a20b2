"""Time the 2D SL step kernel on one F-step of a 2D bench config's fine level:
all intervals' rows at once, as the fused FC phase launches them.  Each extra
argument is a label for one timed run (the launch-bound / record-prefetch
variants were compared this way by rebuilding with an environment switch,
see the note above sl2d_kernel in step2d.cu).
Usage: python tools/sl2d_variants.py cfg4 [label ...]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2203_13382_b200 as P  # noqa: E402
from paper_2203_13382_b200 import mgrit as M  # noqa: E402

name = sys.argv[1]
cfg = P.SolverConfig(**bench.CONFIGS[name])
levels = P.build_hierarchy(cfg)
fine = levels[0]
n = fine.grid.n_points
m = fine.cf
B = cfg.n_t // m
U = torch.empty((cfg.n_t + 1, n), dtype=torch.float64, device="cuda")
U[0] = 0.5
M.pcg64_uniform(cfg.seed, cfg.n_t, n, U[1:])
out = torch.empty((B, n), dtype=torch.float64, device="cuda")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ref = None
for var in sys.argv[2:]:
    os.environ["MGRIT_SL2D_VARIANT"] = var
    for step in range(m - 1):
        fine._apply(U, step, m, B, out)
    torch.cuda.synchronize()
    ts = []
    for rep in range(3):
        e0.record()
        for step in range(m - 1):
            fine._apply(U, step, m, B, out, G=None)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / (m - 1))
    res = out.clone()
    same = ref is None or torch.equal(res, ref)
    ref = res if ref is None else ref
    nodes = B * n
    ms = min(ts)
    print(f"{name} variant {var}: {ms:.3f} ms per batched step ({B} rows), {nodes / ms / 1e6:.3g} Gnode/s, "
          f"bitwise equal to first: {same}")
