"""Time-parallel MGRIT across ranks (one process per GPU).

The time axis of every level is split into contiguous blocks of whole
C-intervals; rank r owns intervals [r*I/P, (r+1)*I/P) of a level with
I = n_steps/m intervals, i.e. the state rows of global steps
[r*I/P*m, (r+1)*I/P*m] (its left boundary C-point included).  Because
n_steps(l+1) = I(l), the coarse level's rank-r rows are exactly the fine
level's C-indices of rank r, so restriction (Gc = R[::m]) and injection
(U[::m] += Uc) never cross ranks.

The only data that moves per sharded level and V-cycle:
  * after F+C relaxation: the C-point buffer row at the block's right edge
    goes to the right neighbour (its F-relaxation starts there);
  * after injection + F-relaxation: the freshly injected left-edge C-point row
    goes to the left neighbour (it is that rank's right edge).
One state row each (8 n bytes), NCCL send/recv over NVLink.  The
convergence norm all-gathers the per-interval partial sums and every rank
adds them in global interval order, so histories are bitwise independent
of P.

A coarse level whose interval count I does not divide by P is split over
Q = gcd(I, Q_finer) rank GROUPS instead of being replicated: the P ranks
form Q groups of P/Q consecutive ranks, every rank of group w owns
intervals [w I/Q, (w+1) I/Q) (the group's members compute them
redundantly), and the row exchanges go between counterpart ranks of
neighbouring groups (rank r <-> r +- P/Q).  Since Q divides the finer
level's group count, a rank's finer C-indices always lie inside its
group's coarse range, so injection stays rank-local; the restriction is
all-gathered once per V-cycle (one C-residual slab per group).  Only the
coarsest level (Q = 1) is fully replicated.  This matters where coarse
levels are bandwidth-bound batched solves (2D, config 5: level 2 has 4
intervals, so at P = 8 each group of 2 ranks solves 1 of them instead of
every rank solving all 4).

The engine is written against a small backend interface (``phase``,
``sweep``, ``total``) so the same sharding / exchange logic runs on the
CUDA kernels (``CudaPhaseBackend``, product) and, in the CPU test-suite, on
a numpy restatement of the phase semantics over gloo.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist

from . import _lib


# ---------------------------------------------------------------------------
# communication


class Comm:
    """Neighbour shifts and all-gathers over a torch.distributed group.

    With NCCL the device rows move directly over NVLink.  ``host_staged``
    routes them through host memory instead, which lets the gloo backend
    drive the CUDA engine (used to test several ranks on one GPU)."""

    def __init__(self, group=None, host_staged: bool | None = None):
        self.group = group
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.size = dist.get_world_size(group) if dist.is_initialized() else 1
        if host_staged is None:
            host_staged = dist.is_initialized() and dist.get_backend(group) != "nccl"
        self.host_staged = host_staged

    def _global(self, r):
        return dist.get_global_rank(self.group, r) if self.group is not None else r

    def shift(self, send: torch.Tensor | None, recv: torch.Tensor | None, direction: int, stride: int = 1):
        """direction=+1: rank r sends to r+stride and receives from r-stride;
        -1 reverses (stride = ranks per group of a group-sharded level)."""
        if self.size == 1:
            return
        ops = []
        dst, src = self.rank + direction * stride, self.rank - direction * stride
        has_send = send is not None and 0 <= dst < self.size
        has_recv = recv is not None and 0 <= src < self.size
        s_buf = send.cpu() if (has_send and self.host_staged and send.is_cuda) else send
        r_buf = torch.empty_like(recv, device="cpu") if (has_recv and self.host_staged and recv.is_cuda) else recv
        if has_send:
            ops.append(dist.P2POp(dist.isend, s_buf, self._global(dst), self.group))
        if has_recv:
            ops.append(dist.P2POp(dist.irecv, r_buf, self._global(src), self.group))
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()
        if has_recv and r_buf is not recv:
            recv.copy_(r_buf)

    def allgather(self, full: torch.Tensor, local: torch.Tensor):
        if self.size == 1:
            full.copy_(local)
            return
        if self.host_staged and full.is_cuda:
            parts = [torch.empty_like(local, device="cpu") for _ in range(self.size)]
            dist.all_gather(parts, local.contiguous().cpu(), group=self.group)
            full.copy_(torch.cat(parts).reshape(full.shape))
            return
        dist.all_gather_into_tensor(full, local.contiguous(), group=self.group)

    def allgather_groups(self, full: torch.Tensor, local: torch.Tensor, stride: int):
        """All-gather when consecutive blocks of `stride` ranks hold identical
        slabs (one group): `full` receives one slab per group, in group order."""
        if stride == 1:
            self.allgather(full, local)
            return
        tmp = torch.empty((self.size,) + tuple(local.shape), dtype=local.dtype, device=local.device)
        self.allgather(tmp.view(self.size * local.shape[0], *local.shape[1:]), local)
        full.copy_(tmp[::stride].reshape(full.shape))


# ---------------------------------------------------------------------------
# plan


@dataclass
class LevelPlan:
    n_steps: int
    m: int | None          # coarsening factor toward the next level (None: coarsest)
    sharded: bool          # split over groups > 1 rank groups (row exchanges needed)
    cb: int = 0            # first owned interval of this rank's group
    ce: int = 0            # one past the last owned interval
    row0: int = 0          # global step of local row 0
    groups: int = 1        # Q: rank groups the level is split over (P: fully sharded, 1: replicated)
    stride: int = 1        # P / Q: ranks per group = rank distance between counterparts

    @property
    def n_intervals(self):
        return self.n_steps // self.m if self.m else 0

    @property
    def local_rows(self):
        return (self.ce - self.cb) * self.m + 1 if self.m else self.n_steps + 1


def make_plan(sizes: list[int], factors: list[int | None], rank: int, size: int) -> list[LevelPlan]:
    """Split level l's I_l intervals over Q_l = gcd(I_l, Q_{l-1}) rank groups
    (Q_{-1} = P): Q = P shards a level fully, 1 < Q < P splits it over groups
    of P/Q ranks, Q = 1 (and always the coarsest level) replicates it.  Q_l
    divides Q_{l-1}, so each rank's finer C-indices lie in its coarse range."""
    plans = []
    q_prev = size
    for N, m in zip(sizes, factors):
        if m is None:
            plans.append(LevelPlan(N, None, False, 0, 0, 0, 1, size))
            continue
        I = N // m
        q = math.gcd(I, q_prev)
        stride = size // q
        w = rank // stride
        cb, ce = w * I // q, (w + 1) * I // q
        plans.append(LevelPlan(N, m, q > 1, cb, ce, cb * m, q, stride))
        q_prev = q
    return plans


# ---------------------------------------------------------------------------
# CUDA backend (product)


class CudaPhaseBackend:
    """Launches the fused phase kernels / sweep of libmgrit_b200.so."""

    # a 2D FC phase can be told that its F-points are already relaxed
    # (mgrit_phase_args::f_relaxed); see TimeParallelCycle.skip_f
    supports_f_relaxed = True

    def __init__(self, levels):
        from .mgrit import _WS
        self.levels = levels
        self.lib = _lib.load()
        self.descs = [lv.desc() for lv in levels[:-1]]
        self.desc_last = levels[-1].desc(stencil_numba=levels[-1].stencil_numba)
        dev = levels[0].device
        need = 0
        for lv, d in zip(levels[:-1], self.descs):
            rows = min(lv.n_steps // lv.cf, max(1, int(self.lib.mgrit_resident_rows(ctypes.byref(d)))))
            need = max(need, int(self.lib.mgrit_gmres_scratch_bytes(ctypes.byref(d), rows)))
        need = max(need, int(self.lib.mgrit_gmres_scratch_bytes(ctypes.byref(self.desc_last), 1)))
        self.scratch = torch.empty(max(need, 8), dtype=torch.uint8, device=dev)
        self.status = _WS.get_status(dev)

    @staticmethod
    def _stream():
        return torch.cuda.current_stream().cuda_stream

    def phase(self, li, phase, *, m, c_begin, c_count, n_intervals, U, u_row0, G, g_row0, Cbuf, Uc, Gc,
              c_row0, partial, partial0, zero_init, f_relaxed=0):
        a = _lib.PhaseArgs()
        n = self.levels[li].grid.n_points
        a.phase, a.m = phase, m
        a.c_begin, a.c_count, a.n_intervals = c_begin, c_count, n_intervals
        a.U, a.ldu, a.u_row0 = U.data_ptr(), n, u_row0
        a.G, a.ldg, a.g_row0 = (0 if G is None else G.data_ptr()), n, g_row0
        a.Cbuf = Cbuf.data_ptr()
        a.Uc = 0 if Uc is None else Uc.data_ptr()
        a.Gc = 0 if Gc is None else Gc.data_ptr()
        a.c_row0 = c_row0
        a.partial = 0 if partial is None else partial.data_ptr()
        a.partial0 = partial0
        a.zero_init = int(zero_init)
        a.f_relaxed = int(f_relaxed)
        rc = self.lib.mgrit_level_phase(ctypes.byref(self.descs[li]), ctypes.byref(a), self.scratch.data_ptr(),
                                        self.scratch.numel(), self.status.data_ptr(), self._stream())
        _lib.check(rc, "level_phase")

    def sweep(self, li, U, G, zero_init):
        n = self.levels[li].grid.n_points
        rc = self.lib.mgrit_sequential_sweep(ctypes.byref(self.desc_last), U.data_ptr(), n,
                                             0 if G is None else G.data_ptr(), n, int(zero_init), 0,
                                             self.scratch.data_ptr(), self.scratch.numel(),
                                             self.status.data_ptr(), self._stream())
        _lib.check(rc, "sequential_sweep")

    def total(self, x: torch.Tensor, out: torch.Tensor):
        _lib.check(self.lib.mgrit_sum(x.data_ptr(), x.numel(), out.data_ptr(), self._stream()), "sum")

    def bad(self) -> bool:
        return int(self.status.item()) != 0


# ---------------------------------------------------------------------------
# engine


class TimeParallelCycle:
    """Buffers and launch/exchange sequence of one sharded V-cycle."""

    def __init__(self, plans: list[LevelPlan], n_points: int, backend, comm: Comm, relaxation: str,
                 U0: torch.Tensor, device, dtype=torch.float64):
        self.plans, self.n, self.be, self.comm, self.relax = plans, n_points, backend, comm, relaxation
        L = len(plans)
        z = lambda rows: torch.zeros((rows, n_points), dtype=dtype, device=device)  # noqa: E731
        self.U = [U0] + [z(p.local_rows) for p in plans[1:]]
        self.G = [None] + [z(p.local_rows) for p in plans[1:]]
        self.C = [z(p.ce - p.cb + 1) for p in plans[:-1]]
        # restriction target of a level whose child is split differently (fewer
        # groups, or replicated): a local slab (row 0 unused), all-gathered
        # per group into the child's rows 1..N_child, then the child's range
        self.Gslab = [None] * L
        self.Gfull = [None] * L
        for li in range(L - 1):
            p, c = plans[li], plans[li + 1]
            if p.groups != c.groups:
                self.Gslab[li] = z(p.ce - p.cb + 1)
                if not (c.groups == 1 and p.stride == 1):
                    self.Gfull[li] = z(c.n_steps)
        p0 = plans[0]
        self.partial = torch.zeros(p0.ce - p0.cb, dtype=dtype, device=device)
        self.partial_all = torch.zeros(p0.n_intervals, dtype=dtype, device=device)
        self.sumsq = torch.zeros(1, dtype=dtype, device=device)
        # As in mgrit._FusedCycle: a V-cycle ends with the fine F-relaxation the
        # next one would start with (same C-points: a rank's F-points depend on
        # its own left C-points only, the row received from the right neighbour
        # is an interval's right end), so the fine 2D FC phase runs only its
        # C-step once prologue() has F-relaxed the rank's intervals.
        lv = getattr(backend, "levels", None)
        self.skip_f = bool(getattr(backend, "supports_f_relaxed", False) and relaxation == "FCF" and L > 1
                           and plans[0].m is not None and lv is not None and lv[0].grid.dim == 2)

    def prologue(self):
        if self.skip_f:
            self.be.phase(0, _lib.PHASE_FC, **self._args(0, _lib.PHASE_FC, False))

    def _args(self, li, phase, zero_init):
        p, c = self.plans[li], self.plans[li + 1]
        Gc = None
        if phase in (_lib.PHASE_F_RES, _lib.PHASE_FONLY_RES):
            Gc = self.Gslab[li] if self.Gslab[li] is not None else self.G[li + 1]
        # the child's U/G local row 0 is global C-index c.row0 (== p.cb when both
        # are split alike, the child group's first step otherwise); Uc is
        # indexed from p.cb, which lies in the child's range
        Uc = self.U[li + 1][p.cb - c.row0:]
        return dict(m=p.m, c_begin=p.cb, c_count=p.ce - p.cb, n_intervals=p.n_intervals, U=self.U[li],
                    u_row0=p.row0, G=self.G[li], g_row0=p.row0, Cbuf=self.C[li], Uc=Uc, Gc=Gc, c_row0=p.cb,
                    partial=self.partial if (li == 0 and phase == _lib.PHASE_INJ_F) else None, partial0=p.cb,
                    zero_init=zero_init)

    def cycle(self, li: int = 0):
        plans, be, comm = self.plans, self.be, self.comm
        p = plans[li]
        zero = li > 0
        if p.m is None:
            be.sweep(li, self.U[li], self.G[li], zero_init=zero)
            return
        last_local = p.ce - p.cb
        if self.relax == "FCF":
            if li == 0 and self.skip_f:
                be.phase(li, _lib.PHASE_FC, f_relaxed=1, **self._args(li, _lib.PHASE_FC, zero))
            else:
                be.phase(li, _lib.PHASE_FC, **self._args(li, _lib.PHASE_FC, zero))
            if p.sharded:
                comm.shift(self.C[li][last_local], self.C[li][0], +1, p.stride)
            be.phase(li, _lib.PHASE_F_RES, **self._args(li, _lib.PHASE_F_RES, zero))
        else:
            be.phase(li, _lib.PHASE_FONLY_RES, **self._args(li, _lib.PHASE_FONLY_RES, zero))
            if p.sharded:
                comm.shift(self.C[li][last_local], self.C[li][0], +1, p.stride)
        if self.Gslab[li] is not None:
            self._gather_restriction(li)
        self.cycle(li + 1)
        be.phase(li, _lib.PHASE_INJ_F, **self._args(li, _lib.PHASE_INJ_F, False))
        if p.sharded:
            comm.shift(self.U[li][0], self.U[li][(p.ce - p.cb) * p.m], -1, p.stride)

    def _gather_restriction(self, li: int):
        """Child forcing rows from every group's C-residual slab."""
        p, c = self.plans[li], self.plans[li + 1]
        slab = self.Gslab[li][1:]
        if self.Gfull[li] is None:        # fully sharded parent, replicated child
            self.comm.allgather(self.G[li + 1][1:], slab)
            return
        full = self.Gfull[li]             # global child steps 1..N_child
        self.comm.allgather_groups(full, slab, p.stride)
        self.G[li + 1][1:].copy_(full[c.row0: c.row0 + c.local_rows - 1])

    def iteration(self):
        """One V-cycle, then the fine residual norm^2 (global order) into sumsq."""
        self.cycle(0)
        self.comm.allgather_groups(self.partial_all, self.partial, self.plans[0].stride)
        self.be.total(self.partial_all, self.sumsq)


def pcg_state_after(seed: int, draws: int):
    """numpy PCG64 state (state, inc) of default_rng(seed) advanced by `draws` steps."""
    st = np.random.default_rng(seed).bit_generator.state["state"]
    state, inc = int(st["state"]), int(st["inc"])
    M = (2549297995355413924 << 64) | 4865540595714422341
    mask = (1 << 128) - 1
    cur_m, cur_p, acc_m, acc_p, d = M, inc, 1, 0, draws
    while d:
        if d & 1:
            acc_m = (acc_m * cur_m) & mask
            acc_p = (acc_p * cur_m + cur_p) & mask
        cur_p = ((cur_m + 1) * cur_p) & mask
        cur_m = (cur_m * cur_m) & mask
        d >>= 1
    return (acc_m * state + acc_p) & mask, inc


def local_rows(cfg, levels, comm: Comm | None = None) -> tuple[int, int]:
    """(first global step, row count) of this rank's fine-level state rows."""
    comm = comm or Comm()
    sizes = [lv.n_steps for lv in levels]
    factors = [lv.cf for lv in levels[:-1]] + [None]
    p0 = make_plan(sizes, factors, comm.rank, comm.size)[0]
    return p0.row0, p0.local_rows


def solve_time_parallel(cfg, levels, comm: Comm | None = None, *, use_graph: bool = True,
                        iterate0=None, out=None):
    """MGRIT solve with the time axis sharded over the ranks of ``comm``.

    ``iterate0``: optional host tensor with this rank's initial-iterate rows
    (global steps max(row0, 1) .. row0 + local_rows - 1); default: numpy's
    PCG64 stream generated on the device from the matching offset.
    ``out``: optional host tensor (local_rows, n_points) receiving the rows.
    Returns (ConvergenceReport, local U rows, LevelPlan of the fine level).
    Identical iterates and bitwise-identical residual histories for any P.
    """
    import time
    from .core import stream_ptr
    from .mgrit import ConvergenceReport, _capture, initial_state

    comm = comm or Comm()
    dev = levels[0].device
    t0 = time.perf_counter()
    sizes = [lv.n_steps for lv in levels]
    factors = [lv.cf for lv in levels[:-1]] + [None]
    plans = make_plan(sizes, factors, comm.rank, comm.size)
    p0 = plans[0]
    n = levels[0].grid.n_points
    U = torch.empty((p0.local_rows, n), dtype=torch.float64, device=dev)
    # local rows = global steps row0 .. row0 + local_rows - 1; iterate draws start at global row 1
    first = p0.row0
    if first == 0:
        U[0] = torch.from_numpy(initial_state(cfg, levels[0].grid)).to(dev)
        rows, start = U[1:], 0
    else:
        rows, start = U, (first - 1) * n
    if iterate0 is not None:
        rows.copy_(torch.as_tensor(iterate0).reshape(rows.shape), non_blocking=True)
    else:
        st, inc = pcg_state_after(cfg.seed, start)
        m64 = (1 << 64) - 1
        _lib.check(_lib.load().mgrit_pcg64_fill(st >> 64, st & m64, inc >> 64, inc & m64, rows.numel(),
                                                int(cfg.iterate == "pm1"), rows.data_ptr(), stream_ptr()),
                   "pcg64")
    be = CudaPhaseBackend(levels)
    be.status.zero_()
    # initial residual over the owned steps (row0+1 .. row0+local_rows-1)
    nloc = p0.local_rows - 1
    row_ss = torch.empty(nloc, dtype=torch.float64, device=dev)
    # only the per-row sums of squares are produced (out = NULL: no residual rows)
    levels[0]._apply(U, p0.row0, 1, nloc, None, U_sub=U[1:], row_sumsq=row_ss)
    row_all = torch.empty(cfg.n_t, dtype=torch.float64, device=dev)
    comm.allgather_groups(row_all, row_ss, p0.stride)
    s0 = torch.zeros(1, dtype=torch.float64, device=dev)
    be.total(row_all, s0)
    r0 = float(torch.sqrt(s0).item())
    eng = TimeParallelCycle(plans, n, be, comm, cfg.relaxation, U, dev)
    eng.prologue()
    hist, state, graph = [r0], "max_iters", None
    for it in range(cfg.max_iters):
        if graph is not None:
            graph.replay()
        else:
            eng.iteration()
            if use_graph and comm.size == 1 and it == 0 and cfg.max_iters > 1:
                graph = _capture(eng.iteration)
        r = float(torch.sqrt(eng.sumsq).item())
        if be.bad():
            hist.append(float("nan"))
            state = "diverged"
            break
        hist.append(r)
        if not np.isfinite(r) or r >= cfg.divergence_factor * r0:
            state = "diverged"
            break
        if r <= cfg.rtol * r0:
            state = "converged"
            break
    if out is not None:
        out.copy_(U)
    torch.cuda.synchronize()
    h = np.array(hist)
    fac = float(h[-1] / h[-2]) if len(h) > 1 else float("nan")
    wall = time.perf_counter() - t0
    return ConvergenceReport(h, len(h) - 1, state, fac, wall, 0.0, wall), U, p0


# ---------------------------------------------------------------------------
# sharded hierarchy construction


def build_hierarchy_sharded(cfg, comm: Comm | None = None):
    """``build_hierarchy`` (mgrit.py:217-269) for a time-sharded solve.

    Every rank traces (ERK), backtracks and computes sigma only for the steps
    its rank group works on: on level l the steps of the group's intervals,
    all steps on the replicated coarsest level.  Coarse step c of level l is
    interval c of level l-1, so the rank that owns that interval holds its m
    children and builds the step locally; where level l is split over fewer
    groups than level l-1 (or replicated) the built slabs are all-gathered
    (``Comm.allgather_groups``) and the group's range is kept.  Records are
    bit-identical to the replicated build's (same kernels on the same data)
    and per-rank record memory drops from all n_t fine steps to n_t / P.
    A level stores steps [set0, set0 + S_local); the kernels address the
    stored rows through the level descriptor (``Level.desc``)."""
    from . import mgrit as M
    from .core import Grid1D, Grid2D, require_cuda, stream_ptr

    comm = comm or Comm()
    speed = cfg.speed
    if comm.size == 1 or speed.constant or cfg.operator_kind == "ideal":
        return M.build_hierarchy(cfg)     # one shared record set / composed operator: nothing to shard
    if cfg.departure_policy != "backtrack":
        return M.build_hierarchy(cfg)
    dev = require_cuda()
    grid = Grid1D(cfg.n_x) if cfg.dim == 1 else Grid2D(cfg.n_x)
    n = grid.n_points
    dt = cfg.dt if cfg.dt is not None else M.DEFAULT_CFL * grid.h
    lib = _lib.load()
    # level sizes / factors exactly as build_hierarchy derives them
    sizes, factors = [cfg.n_t], []
    while cfg.max_levels is None or len(sizes) < cfg.max_levels:
        m = cfg.schedule_factor(len(sizes) - 1)
        if sizes[-1] % m != 0 or sizes[-1] // m < 2:
            break
        factors.append(m)
        sizes.append(sizes[-1] // m)
    if len(sizes) < 2:
        raise ValueError("time grid does not admit any coarsening with the given schedule")
    factors.append(None)
    plans = make_plan(sizes, factors, comm.rank, comm.size)

    def need(li):
        p = plans[li]
        return (0, p.n_steps) if p.m is None else (p.cb * p.m, p.ce * p.m)

    def rows(t, first):          # pointer to stored row `first` of a (S, n) tensor (0 if absent)
        return 0 if t is None else t.data_ptr() + first * n * 8

    a, b = need(0)
    s_x, s_y, d_x, d_y = M._erk(grid, speed, cfg.erk_order, b - a, dt, 1, dt, dev, set_first=a)
    fine = M.Level(0, grid, cfg.p, cfg.n_t, dt, "fine", s_x, s_y, d_x, d_y, set0=a)
    levels = [fine]
    for li in range(1, len(sizes)):
        prev, pp, m = levels[-1], plans[li - 1], factors[li - 1]
        c0, c1 = pp.cb, pp.ce                       # coarse steps whose children this rank holds
        cnt = c1 - c0
        off = c0 * m - prev.set0                    # first child's stored row
        s_x, s_y, d_x, d_y = M._alloc_records(cnt, n, grid.dim, dev)
        _lib.check(lib.mgrit_backtrack(grid.dim, grid.n_x, m, cnt, 0, rows(prev.disp_x, off),
                                       rows(prev.disp_y, off), s_x.data_ptr(), M._ptr(s_y), d_x.data_ptr(),
                                       M._ptr(d_y), stream_ptr()), "backtrack")
        sig_x = sig_y = None
        if cfg.operator_kind in ("corrected", "forward_euler"):
            sig_x = torch.empty((cnt, n), dtype=torch.float64, device=dev)
            sig_y = torch.empty_like(sig_x) if grid.dim == 2 else None
            _lib.check(lib.mgrit_phi_sigma(grid.dim, grid.n_x, cfg.p, m, cnt, 0, s_x.data_ptr(), M._ptr(s_y),
                                           rows(prev.s_x, off), rows(prev.s_y, off), rows(prev.sig_x, off),
                                           rows(prev.sig_y, off), sig_x.data_ptr(), M._ptr(sig_y), stream_ptr()),
                       "phi_sigma")
        a, b = need(li)
        if (a, b) != (c0, c1):
            # the level is split over fewer groups than its parent: gather every
            # group's slab (one per parent group, in order), keep this group's range
            def gather(t):
                if t is None:
                    return None
                full = torch.empty((sizes[li], n), dtype=torch.float64, device=dev)
                comm.allgather_groups(full, t, pp.stride)
                return full[a:b].clone()
            s_x, s_y, d_x, d_y, sig_x, sig_y = (gather(t) for t in (s_x, s_y, d_x, d_y, sig_x, sig_y))
        lvl = M.Level(li, grid, cfg.p, sizes[li], prev.dt * m, cfg.operator_kind, s_x, s_y, d_x, d_y, sig_x, sig_y,
                      finer=prev, set0=a)
        prev.cf = m
        prev.disp_x = prev.disp_y = None
        levels.append(lvl)
    levels[-1].disp_x = levels[-1].disp_y = None
    mode = cfg.gmres_mode or ("fixed" if len(levels) == 2 else "tolerance")
    gcfg = M.GmresConfig(10, None if mode == "fixed" else 1e-2, cfg.gmres_variant)
    for lvl in levels[1:]:
        lvl.gmres_cfg = gcfg
    last = levels[-1]
    last.stencil_numba = (last.grid.dim == 1 and last.kind == "corrected" and last.n_steps >= 64)
    return levels
