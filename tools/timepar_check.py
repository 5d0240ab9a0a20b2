"""Time-sharded solve of a full-size bench config with P ranks on ONE GPU
(gloo, rows staged through host memory) against the single-rank solve:
iteration count, residual history and the whole space-time iterate must be
bit-identical.  This exercises the exact partition (interval blocks, group
splits of coarse levels, row exchanges, grouped all-gathers) that P GPUs
would run; the NCCL transport itself needs P GPUs.  Tools only.

    python tools/timepar_check.py cfg2 8 [launch_policy]
"""
import json
import os
import socket
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, size, port, name, out, policy):
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=size)
    try:
        import bench
        import paper_2203_13382_b200 as P
        from paper_2203_13382_b200 import timepar as T
        P.set_launch_policy(policy)
        cfg = P.SolverConfig(**bench.CONFIGS[name])
        levels = P.build_hierarchy(cfg)
        comm = T.Comm()
        plan = T.make_plan([lv.n_steps for lv in levels], [lv.cf for lv in levels[:-1]] + [None],
                           comm.rank, comm.size)
        rep, U, p0 = T.solve_time_parallel(cfg, levels, comm)
        rows = U[1:].cpu()
        sizes = [torch.zeros(1, dtype=torch.int64) for _ in range(size)]
        dist.all_gather(sizes, torch.tensor([rows.shape[0]], dtype=torch.int64))
        allr = [torch.empty((int(s.item()), rows.shape[1]), dtype=rows.dtype) for s in sizes]
        dist.all_gather(allr, rows)
        if rank == 0:
            full = torch.cat([U[:1].cpu()] + allr).numpy()
            np.savez(out, U=full, hist=rep.residual_norms, iters=rep.iterations,
                     groups=np.array([lp.groups for lp in plan]))
    finally:
        dist.destroy_process_group()


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
    ranks = int(sys.argv[2]) if len(sys.argv) > 2 else 4
    policy = sys.argv[3] if len(sys.argv) > 3 else "auto"
    import bench
    import paper_2203_13382_b200 as P
    P.set_launch_policy(policy)
    out = f"/tmp/timepar_{name}_{ranks}.npz"
    t0 = time.perf_counter()
    mp.spawn(_worker, args=(ranks, _free_port(), name, out, policy), nprocs=ranks, join=True)
    t_sharded = time.perf_counter() - t0
    got = np.load(out)
    cfg = P.SolverConfig(**bench.CONFIGS[name])
    rep, U = P.solve(cfg)
    r0 = rep.residual_norms[0]
    n_common = min(len(got["hist"]), len(rep.residual_norms))
    res = {"config": name, "ranks": ranks, "launch_policy": policy,
           "transport": "gloo, rows staged through host (one GPU)",
           "iterations": int(got["iters"]), "single_rank_iterations": rep.iterations,
           "history_bitwise_equal": bool(np.array_equal(got["hist"], rep.residual_norms)),
           "iterate_bitwise_equal": bool(np.array_equal(got["U"], U)),
           "max_history_dev_over_r0": float(np.max(np.abs(got["hist"][:n_common] - rep.residual_norms[:n_common])) / r0),
           "iterate_rel_dev": float(np.linalg.norm(got["U"] - U) / np.linalg.norm(U)),
           "final_residual_over_r0": float(rep.residual_norms[-1] / rep.residual_norms[0]),
           "groups_per_level": [int(g) for g in got["groups"]],
           "wall_s_including_setup": round(t_sharded, 1)}
    print(json.dumps(res))


if __name__ == "__main__":
    main()
