"""Run one fused level phase of a bench config between cudaProfilerStart/Stop,
so that `ncu --profile-from-start off --metrics dram__bytes_read.sum,...`
sees exactly the launches bench.py times as that phase (tools only).

Usage: python tools/profile_phase.py cfg4 L1_F_RES_corrected
The key is bench.py's kernel_breakdown name: L<level>_<FC|F_RES|FONLY_RES|INJ_F>_<kind>.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2203_13382_b200 as P  # noqa: E402
from paper_2203_13382_b200 import _lib  # noqa: E402
from paper_2203_13382_b200 import mgrit as M  # noqa: E402

name, key = sys.argv[1], sys.argv[2]
li = int(key.split("_")[0][1:])
ph_name = key.split("_", 1)[1].rsplit("_", 1)[0]
phase = {"FC": _lib.PHASE_FC, "F_RES": _lib.PHASE_F_RES, "FONLY_RES": _lib.PHASE_FONLY_RES,
         "INJ_F": _lib.PHASE_INJ_F}[ph_name]
cfg = P.SolverConfig(**bench.CONFIGS[name])
levels = P.build_hierarchy(cfg)
n = levels[0].grid.n_points
U = torch.empty((cfg.n_t + 1, n), dtype=torch.float64, device="cuda")
U[0] = torch.from_numpy(M.initial_state(cfg, levels[0].grid)).cuda()
M.pcg64_uniform(cfg.seed, cfg.n_t, n, U[1:])
eng = M._FusedCycle(levels, U, cfg.relaxation)
eng.prologue()
eng.iteration()                      # every buffer holds the state of a real V-cycle
eng._phase(li, phase)                # warm (first-launch attributes)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
eng._phase(li, phase)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("profiled", name, key)
