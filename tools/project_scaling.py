"""Per-rank compute time of the time-sharded V-cycle at P ranks, measured on
ONE GPU (tools only; a projection, not a multi-GPU measurement).

Rank r's kernels of one V-cycle run exactly as in solve_time_parallel, but
the communicator is a local stub: neighbour rows are not exchanged and the
all-gathers replicate the local slab, so the values (and hence tolerance-
mode GMRES counts) drift from a real run; the V-cycle's launch sequence and
per-rank sizes are the real ones.  The NVLink traffic of the real run is
counted from the plan and added at a stated bandwidth.

    python tools/project_scaling.py cfg5 [P ...]
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2203_13382_b200 as P  # noqa: E402
from paper_2203_13382_b200 import _lib  # noqa: E402
from paper_2203_13382_b200 import mgrit as M  # noqa: E402
from paper_2203_13382_b200 import timepar as T  # noqa: E402

NVLINK_GBS = 700.0   # achievable per-direction NVLink 5 bandwidth assumed for the exchange term


class StubComm:
    def __init__(self, rank, size):
        self.rank, self.size, self.bytes = rank, size, 0
        self.host_staged = False

    def shift(self, send, recv, direction, stride=1):
        dst, src = self.rank + direction * stride, self.rank - direction * stride
        if send is not None and 0 <= dst < self.size:
            self.bytes += send.numel() * send.element_size()

    def allgather(self, full, local):
        k = full.numel() // local.numel()
        full.view(k, -1).copy_(local.reshape(1, -1).expand(k, -1))
        self.bytes += (self.size - 1) * local.numel() * local.element_size()

    def allgather_groups(self, full, local, stride):
        self.allgather(full, local)


def per_rank_ms(cfg, levels, rank, size, iters=3):
    sizes = [lv.n_steps for lv in levels]
    factors = [lv.cf for lv in levels[:-1]] + [None]
    plans = T.make_plan(sizes, factors, rank, size)
    p0 = plans[0]
    n = levels[0].grid.n_points
    dev = levels[0].device
    U = torch.empty((p0.local_rows, n), dtype=torch.float64, device=dev)
    M.pcg64_uniform(cfg.seed, p0.local_rows, n, U)
    comm = StubComm(rank, size)
    be = T.CudaPhaseBackend(levels)
    eng = T.TimeParallelCycle(plans, n, be, comm, cfg.relaxation, U, dev)
    eng.prologue()
    eng.iteration()
    torch.cuda.synchronize()
    comm.bytes = 0
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters):
        eng.iteration()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / iters, comm.bytes / iters, [p.groups for p in plans]


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "cfg5"
    Ps = [int(x) for x in sys.argv[2:]] or [1, 2, 4, 8]
    cfg = P.SolverConfig(**bench.CONFIGS[name])
    levels = P.build_hierarchy(cfg)
    out = {"config": name, "nvlink_gbs_assumed": NVLINK_GBS, "per_P": {}}
    for size in Ps:
        # the slowest rank bounds the step: time ranks 0 (left edge) and P-1
        ranks = sorted({0, size - 1})
        worst = 0.0
        for r in ranks:
            ms, nbytes, groups = per_rank_ms(cfg, levels, r, size)
            comm_ms = nbytes / (NVLINK_GBS * 1e9) * 1e3
            worst = max(worst, ms + comm_ms)
            out["per_P"].setdefault(str(size), {})[f"rank{r}"] = {
                "compute_ms_per_iteration": round(ms, 3), "exchange_MB_per_iteration": round(nbytes / 1e6, 2),
                "exchange_ms_at_assumed_bw": round(comm_ms, 3), "groups_per_level": groups}
        out["per_P"][str(size)]["projected_ms_per_iteration"] = round(worst, 3)
    base = out["per_P"][str(Ps[0])]["projected_ms_per_iteration"]
    for size in Ps:
        d = out["per_P"][str(size)]
        d["projected_speedup_vs_P%d" % Ps[0]] = round(base / d["projected_ms_per_iteration"], 2)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
