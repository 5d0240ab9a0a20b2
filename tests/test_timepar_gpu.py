"""Time-parallel CUDA engine with several ranks on one GPU (gloo, rows staged
through host memory): the sharded solve reproduces the single-rank solve
bit-for-bit — same iterates, same residual history — for 1D and 2D."""

import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CASES = {
    "1d_b2_p3_m4": dict(n_x=256, n_t=256, wave_speed="B2", p=3, schedule=4, seed=1),
    "1d_c3_frelax": dict(n_x=128, n_t=128, wave_speed="C3", p=1, schedule=4, relaxation="F"),
    "1d_replicated_tail": dict(n_x=128, n_t=96, wave_speed="C3", p=3, schedule=4),
    "2d_b4_p3_m4": dict(n_x=16, n_t=64, dim=2, wave_speed="B4", p=3, schedule=4, u0="sin4", seed=3),
    # levels [32, 8, 2]: with 4 ranks level 1 (2 intervals) is split over 2
    # rank groups (counterpart exchanges + grouped restriction all-gather)
    "1d_group_split": dict(n_x=128, n_t=32, wave_speed="B2", p=3, schedule=4, seed=1),
    "2d_group_split": dict(n_x=16, n_t=32, dim=2, wave_speed="B4", p=3, schedule=4, u0="sin4", seed=3),
}


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, size, port, kw, out, build="replicated"):
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=size)
    try:
        import paper_2203_13382_b200 as P
        from paper_2203_13382_b200 import timepar as T
        cfg = P.SolverConfig(**kw)
        comm = T.Comm()
        if build == "sharded":
            levels = T.build_hierarchy_sharded(cfg, comm)
            # records of the owned steps only (1/P of the fine level)
            assert levels[0].s_x.shape[0] == cfg.n_t // size
        else:
            levels = P.build_hierarchy(cfg)
        rep, U, p0 = T.solve_time_parallel(cfg, levels, comm)
        rows = U[1:].cpu()
        allr = [torch.empty_like(rows) for _ in range(size)]
        dist.all_gather(allr, rows)
        if rank == 0:
            full = torch.cat([U[:1].cpu()] + allr).numpy()
            np.savez(out, U=full, hist=rep.residual_norms, iters=rep.iterations)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name", list(CASES))
@pytest.mark.parametrize("ranks", [2, 4])
@pytest.mark.parametrize("build", ["replicated", "sharded"])
def test_sharded_cuda_engine_equals_single_rank(tmp_path, name, ranks, build):
    """Replicated hierarchy, or the per-rank sharded build (each rank traces /
    backtracks / computes sigma only for its group's steps): both reproduce
    the single-GPU solve bit for bit."""
    import paper_2203_13382_b200 as P
    kw = CASES[name]
    if (kw["n_t"] // kw["schedule"]) % ranks:
        pytest.skip("fine level not divisible")
    out = str(tmp_path / "r.npz")
    mp.spawn(_worker, args=(ranks, _free_port(), kw, out, build), nprocs=ranks, join=True)
    got = np.load(out)
    cfg = P.SolverConfig(**kw)
    rep, U = P.solve(cfg)
    assert int(got["iters"]) == rep.iterations
    assert np.array_equal(got["hist"], rep.residual_norms)
    assert np.array_equal(got["U"], U)
