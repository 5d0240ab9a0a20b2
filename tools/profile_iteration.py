"""Run one eager MGRIT iteration of a bench config between cudaProfilerStart/Stop
(for `ncu --profile-from-start off`).  Usage: python tools/profile_iteration.py [cfg2]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2203_13382_b200 as P  # noqa: E402
from paper_2203_13382_b200 import mgrit as M  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
cfg = P.SolverConfig(**bench.CONFIGS[name])
levels = P.build_hierarchy(cfg)
P.solve(cfg, levels, output="device")            # warm-up (attributes, JIT-free)
n = levels[0].grid.n_points
U = torch.empty((cfg.n_t + 1, n), dtype=torch.float64, device="cuda")
U[0] = torch.from_numpy(M.initial_state(cfg, levels[0].grid)).cuda()
M.pcg64_uniform(cfg.seed, cfg.n_t, n, U[1:])
eng = M._FusedCycle(levels, U, cfg.relaxation)
eng.prologue()
eng.iteration()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
eng.iteration()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("profiled one iteration of", name)
