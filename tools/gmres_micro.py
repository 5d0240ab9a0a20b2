"""Micro-benchmark: one corrected step (SL + fixed-K GMRES) on one CTA vs K.
Usage: python tools/gmres_micro.py [n_x]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2203_13382_b200 as P  # noqa: E402
from paper_2203_13382_b200 import mgrit as M  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
cfg = P.SolverConfig(n_x=n, n_t=256, wave_speed="B2", p=3, schedule=4)
levels = P.build_hierarchy(cfg)
lv = levels[3]


def timeit(fn, reps=10, inner=10):
    """Device time per call: `inner` calls captured in a CUDA graph, replayed."""
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(inner):
            fn()
    g.replay()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3 / inner)
    return float(np.median(ts))


U = torch.from_numpy(np.random.default_rng(0).standard_normal((4, n))).cuda()
out = torch.empty_like(U)
for B in (1, 4):
    res = []
    for K in (1, 2, 3, 5, 8, 10):
        lv.gmres_cfg = M.GmresConfig(K, None)
        res.append((K, timeit(lambda: lv._apply(U, 0, 1, B, out))))
    print(f"n={n} B={B} kind={lv.kind} us per call by K:", " ".join(f"K{K}:{t:.1f}" for K, t in res), flush=True)
fine = levels[0]
print(f"plain SL one row: {timeit(lambda: fine._apply(U, 0, 1, 1, out)):.1f} us", flush=True)
