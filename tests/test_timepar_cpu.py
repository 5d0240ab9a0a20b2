"""Time-parallel engine (paper_2203_13382_b200/timepar.py) on CPU over gloo.

The sharding plan, halo exchanges, restriction/injection index maps and the
global-order norm are exercised with world_size 1 and 2 using the numpy
restatement of the phase kernels (tests/phase_oracle.py).  Contract: the
iterates of every rank count are bit-identical to each other and to the
reference-structured oracle solve, and the residual norms are bit-identical
across rank counts.
"""

import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import oracle as O  # noqa: E402
from paper_2203_13382_b200 import timepar as T  # noqa: E402
from phase_oracle import OraclePhaseBackend  # noqa: E402

CASES = {
    "c3_p3_m4": dict(n_x=32, n_t=64, wave_speed="C3", p=3, schedule=4),
    "b2_p5_m8": dict(n_x=64, n_t=128, wave_speed="B2", p=5, schedule=8, seed=2),
    "replicated_tail": dict(n_x=32, n_t=48, wave_speed="C2", p=1, schedule=4),
    "f_relax": dict(n_x=32, n_t=64, wave_speed="C3", p=1, schedule=4, relaxation="F"),
    "two_level_fixed": dict(n_x=32, n_t=64, wave_speed="C1", p=1, schedule=8, max_levels=2, iterate="pm1"),
}
# levels [32, 8, 2]: at P = 4 the fine level is fully sharded and level 1
# (2 intervals) is split over 2 groups of 2 ranks
GROUP_CASES = {
    "group_split": dict(n_x=32, n_t=32, wave_speed="C3", p=3, schedule=4),
    "group_split_f": dict(n_x=32, n_t=128, wave_speed="B2", p=1, schedule=8, relaxation="F", seed=2),
}
ITERS = 3


def _initial(ocfg):
    U = np.empty((ocfg.n_t + 1, ocfg.n_x))
    U[0] = O.initial_state(ocfg)
    U[1:] = O.initial_iterate(ocfg)
    return U


def run_engine(kw, rank, size):
    ocfg = O.OConfig(**kw)
    levels = O.hierarchy(ocfg)
    sizes = [lv.n_steps for lv in levels]
    factors = [lv.cf for lv in levels[:-1]] + [None]
    plans = T.make_plan(sizes, factors, rank, size)
    p0 = plans[0]
    Ufull = _initial(ocfg)
    U = torch.from_numpy(Ufull[p0.row0: p0.row0 + p0.local_rows].copy())
    eng = T.TimeParallelCycle(plans, ocfg.n_x, OraclePhaseBackend(levels), T.Comm(), ocfg.relaxation, U,
                              torch.device("cpu"))
    norms = []
    for _ in range(ITERS):
        eng.iteration()
        norms.append(float(eng.sumsq.item()))
    return U.numpy(), p0, norms, [p.sharded for p in plans]


def _worker(rank, size, port, kw, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=size)
    try:
        U, p0, norms, sharded = run_engine(kw, rank, size)
        # gather the owned rows (rows row0+1 .. row0+local_rows-1; rank 0 also row 0)
        rows = torch.from_numpy(U[1:].copy())
        allr = [torch.empty_like(rows) for _ in range(size)]
        dist.all_gather(allr, rows)
        if rank == 0:
            full = np.concatenate([U[:1]] + [t.numpy() for t in allr])
            np.savez(out_path, U=full, norms=np.array(norms), sharded=np.array(sharded))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_plan_shards_and_replicates():
    plans = T.make_plan([4096, 1024, 256, 64, 16, 4], [4, 4, 4, 4, 4, None], 3, 8)
    # level 4 has 4 intervals: split over 4 groups of 2 ranks (rank 3 -> group 1)
    assert [p.groups for p in plans] == [8, 8, 8, 8, 4, 1]
    assert [p.sharded for p in plans] == [True, True, True, True, True, False]
    assert (plans[4].stride, plans[4].cb, plans[4].ce, plans[4].row0, plans[4].local_rows) == (2, 1, 2, 4, 5)
    assert (plans[0].cb, plans[0].ce, plans[0].row0, plans[0].local_rows) == (384, 512, 1536, 513)
    # coarse rank-r rows are exactly the fine level's C-indices of rank r
    for f, c in zip(plans[:3], plans[1:4]):
        assert c.row0 == f.cb and c.local_rows == f.ce - f.cb + 1
    # ... and a group-split child's range contains them
    f, c = plans[3], plans[4]
    assert c.row0 <= f.cb and f.ce <= c.row0 + c.local_rows - 1
    one = T.make_plan([64, 16, 4], [4, 4, None], 0, 1)
    assert [p.sharded for p in one] == [False, False, False] and one[0].local_rows == 65
    # cfg5 at P = 8: level 2 (4 intervals) over 4 groups, coarsest replicated
    c5 = T.make_plan([2048, 256, 32, 4], [8, 8, 8, None], 5, 8)
    assert [p.groups for p in c5] == [8, 8, 4, 1] and (c5[2].cb, c5[2].ce) == (2, 3)
    # I not divisible by P: gcd groups (12 intervals over 8 ranks -> 4 groups)
    odd = T.make_plan([48, 12, 3], [4, 4, None], 7, 8)
    assert [p.groups for p in odd] == [4, 1, 1] and (odd[0].cb, odd[0].ce) == (9, 12)


@pytest.mark.parametrize("name", list(CASES))
def test_single_rank_engine_matches_reference_structured_oracle(name):
    kw = CASES[name]
    U, _, norms, _ = run_engine(kw, 0, 1)
    ocfg = O.OConfig(**{**kw, "max_iters": ITERS, "rtol": 0.0})
    rep, Uo = O.solve(ocfg)
    assert np.array_equal(U, Uo), np.max(np.abs(U - Uo))
    r = np.sqrt(np.array(norms))
    assert np.all(np.abs(r - rep.residual_norms[1:]) <= 1e-12 * rep.residual_norms[0])


@pytest.mark.parametrize("name", list(CASES))
def test_two_ranks_gloo_match_one_rank(tmp_path, name):
    kw = CASES[name]
    out = str(tmp_path / "r.npz")
    mp.spawn(_worker, args=(2, _free_port(), kw, out), nprocs=2, join=True)
    got = np.load(out)
    U1, _, norms1, _ = run_engine(kw, 0, 1)
    assert np.array_equal(got["U"], U1)
    assert np.array_equal(got["norms"], np.array(norms1))
    if name == "replicated_tail":
        assert list(got["sharded"]) == [True, False, False]


@pytest.mark.parametrize("name", list(GROUP_CASES))
def test_four_ranks_group_split_match_one_rank(tmp_path, name):
    """A coarse level with fewer intervals than ranks is split over rank
    groups (counterpart exchanges, grouped restriction all-gather): the
    iterates and norms equal the single-rank engine's bit-for-bit."""
    kw = GROUP_CASES[name]
    ocfg = O.OConfig(**kw)
    levels = O.hierarchy(ocfg)
    plans = T.make_plan([lv.n_steps for lv in levels], [lv.cf for lv in levels[:-1]] + [None], 0, 4)
    assert plans[0].groups == 4 and 1 < plans[1].groups < 4
    out = str(tmp_path / "r.npz")
    mp.spawn(_worker, args=(4, _free_port(), kw, out), nprocs=4, join=True)
    got = np.load(out)
    U1, _, norms1, _ = run_engine(kw, 0, 1)
    assert np.array_equal(got["U"], U1)
    assert np.array_equal(got["norms"], np.array(norms1))
