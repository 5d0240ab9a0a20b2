"""Benchmark: MGRIT solve space-time DOF/s to 1e-10 relative residual.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg5] [--impl reference]

One *step* = one complete MGRIT solve (BASELINE.json metric) of the chosen
config from the prebuilt device hierarchy: U initialisation (numpy PCG64
stream generated bit-identically on the device), initial residual, V-cycles
and convergence residuals until ||r|| <= 1e-10 ||r0||.  Hierarchy setup
(ERK tracing, backtracking, sigma) is excluded and reported separately, as in
the reference's timing discussion.

Default workload: BASELINE config 5, the largest configuration that fits one
GPU (configs[4]): 2D, 1024^2 mesh x 2048 steps = 2^31 space-time DOF,
a(x,y,t) = (cos^2(pi x) cos(2 pi t) + 0.5, sin^2(pi y) cos(2 pi t) + 0.5),
p = 5, m = 8 multilevel FCF (levels 2048/256/32/4), u0 = sin^4 sin^4, seed 4,
dt = 0.85 h (reference default).  U (17 GB) and the fine departure records
(34 GB) exceed the 126 MB L2 many times over, so no flush is needed; configs
whose inputs are under twice the L2 (cfg1) get an untimed 256 MiB write
before each timed solve.  ``--config cfg2`` etc. select the other configs.

``--impl reference`` times the reference's CPU implementation of the path —
the oracle port under oracle/ (bit-identical to mgrit_advect; the reference
is pure Python, so there is nothing to compile into oracle/_ref) — on the
host, on the same config/metric:
  * cfg1, cfg2: one V-cycle + convergence residual per step, extrapolated with
    the reference's own iteration count;
  * cfg3-cfg5 (a full V-cycle takes minutes to hours on the CPU): per step one
    full-size fine SL step and one full-size corrected coarse step, then
    cost = r0 + iterations x (applications per V-cycle x per-application
    time), counting the reference's applications exactly (mgrit.py:276-334:
    N(4 - 2/m) per non-coarsest level, N on the coarsest, plus the fine
    convergence residual) — labelled "extrapolated".

N > 1: under torchrun the time axis of the one solve is sharded across the
ranks (paper_2203_13382_b200/timepar.py; NCCL send/recv of boundary C-point
rows, all-gathered norm partials) — strong scaling.  Without torchrun,
``--gpus N`` (N > 1) re-launches itself under torch.distributed.run with N
ranks, one GPU each.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    "cfg1": dict(n_x=1024, n_t=1024, wave_speed="C1", p=1, schedule=8, max_levels=2, dt=2.0 / 1024, seed=0,
                 iterate="pm1"),
    "cfg1_085h": dict(n_x=1024, n_t=1024, wave_speed="C1", p=1, schedule=8, max_levels=2, seed=0, iterate="pm1"),
    "cfg2": dict(n_x=4096, n_t=4096, wave_speed="B2", p=3, schedule=4, seed=1),
    "cfg3": dict(n_x=16384, n_t=16384, wave_speed="B2", p=5, schedule=8, seed=2),
    "cfg4": dict(n_x=512, n_t=1024, dim=2, wave_speed="B4", p=3, schedule=4, seed=3, u0="sin4"),
    "cfg5": dict(n_x=1024, n_t=2048, dim=2, wave_speed="B4", p=5, schedule=8, seed=4, u0="sin4"),
}
DEFAULT_CONFIG = "cfg5"
DESCR = {
    "cfg1": "BASELINE cfg1: 1D a=1, 1024x1024, p=1, two-level m=8, dt=2/nt (CFL 1), iterate U[-1,1) seed 0",
    "cfg1_085h": "BASELINE cfg1 mesh at dt=0.85h (non-degenerate companion)",
    "cfg2": "BASELINE cfg2: 1D a=1+0.5sin(2pi x)cos(2pi t), 4096x4096, p=3, m=4 multilevel FCF, seed 1, dt=0.85h",
    "cfg3": "BASELINE cfg3: 1D same speed, 16384x16384, p=5, m=8 multilevel FCF, seed 2, dt=0.85h",
    "cfg4": "BASELINE cfg4: 2D a=(cos^2(pi x)cos(2pi t)+.5, sin^2(pi y)cos(2pi t)+.5), 512^2 x 1024, p=3, m=4, "
            "u0=sin^4 sin^4, seed 3, dt=0.85h",
    "cfg5": "BASELINE cfg5: 2D same speed, 1024^2 x 2048, p=5, m=8 multilevel FCF, u0=sin^4 sin^4, seed 4, dt=0.85h",
}
# full-size reference histories: index.json solves (real reference) and the
# tests/golden/make_fullsize.py fixtures (cfg4: real reference; cfg3: the
# bit-pinned oracle, the reference does not fit 62 GB)
GOLDEN = {"cfg1": "cfg1_full", "cfg1_085h": "cfg1_085h", "cfg2": "cfg2_full"}
FULLSIZE = {"cfg3": "cfg3_full", "cfg4": "cfg4_full"}
# config 5 has no full-size CPU reference (> 150 GB, hours per V-cycle); its
# mesh/degree/factor/speed/seed/u0 on 128 steps has (real reference, 2 V-cycles)
CFG5_MESH_FIXTURE = "cfg5mesh_nt128"
# iteration counts the reference arm extrapolates with where no full CPU
# solve is feasible: the reference's own count where a full-size fixture
# exists, else the count the GPU solve reaches (histories agree to 1e-12 r0
# wherever both exist)
EXTRAP_ITERS = {"cfg3": (32, "GPU solve (the full-size oracle fixture reproduces it where complete)"),
                "cfg4": (13, "GPU solve (the real reference's full-size fixture reproduces it where complete)"),
                "cfg5": (14, "GPU solve (no CPU reference is feasible at this size)")}

L2_BYTES = 126 * 1024 * 1024   # B200 L2
METRIC = "MGRIT solve space-time DOF/s to 1e-10 residual"


def level_sizes(kw) -> tuple[list[int], list[int | None]]:
    """Level step counts and coarsening factors (mgrit.py:234-244: coarsen
    while N/m >= 2 and m divides N, up to max_levels)."""
    sched = kw["schedule"]
    sizes, factors = [kw["n_t"]], []
    while kw.get("max_levels") is None or len(sizes) < kw["max_levels"]:
        m = sched if isinstance(sched, int) else list(sched)[min(len(sizes) - 1, len(sched) - 1)]
        N = sizes[-1]
        if N % m or N // m < 2:
            break
        factors.append(m)
        sizes.append(N // m)
    return sizes, factors + [None]


def static_config(name: str) -> dict:
    """The workload description both arms print (identical dicts)."""
    kw = CONFIGS[name]
    dim = kw.get("dim", 1)
    sizes, _ = level_sizes(kw)
    npts = kw["n_x"] ** dim
    dt = kw.get("dt") or 0.85 * 2.0 / kw["n_x"]
    rec_sets = 1 if kw["wave_speed"] in ("C1", "C4") else kw["n_t"]
    in_bytes = 8 * (kw["n_t"] + 1) * npts + 8 * dim * npts * rec_sets
    return {"workload": DESCR[name], "name": name, "dim": dim, "n_x": kw["n_x"], "n_t": kw["n_t"],
            "dof": npts * kw["n_t"], "p": kw["p"], "schedule": kw["schedule"], "levels": sizes, "dt": dt,
            "seed": kw["seed"], "u0": kw.get("u0", "reference"), "iterate": kw.get("iterate", "uniform01"),
            "rtol": 1e-10,
            "l2": (f"inputs larger than L2 ({in_bytes / 2**20:.0f} MiB of U + fine departure records "
                   f"> {L2_BYTES / 2**20:.0f} MiB)" if in_bytes >= 2 * L2_BYTES else
                   f"L2 flushed before every timed solve (untimed 256 MiB write; inputs "
                   f"{in_bytes / 2**20:.0f} MiB < 2 x {L2_BYTES / 2**20:.0f} MiB L2)")}


def _dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region.

    Every sample line is stamped with the host clock, so the summary can keep
    only the samples taken between mark("start") and mark("stop").  A timed
    region shorter than a few sampling periods (cfg1: ~4 ms) falls back to the
    samples of the surrounding load (warm-up + an untimed tail of the same
    solves) and says so in "window"."""

    PERIOD_MS = 20

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines: list[tuple[float, str]] = []
        self.marks: dict[str, float] = {}

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", str(self.PERIOD_MS)],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            t_end = time.perf_counter() + 5.0          # wait until nvidia-smi is live
            while not self.lines and time.perf_counter() < t_end and self.proc.poll() is None:
                time.sleep(0.01)
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.perf_counter(), line.strip()))

    def mark(self, name: str):
        self.marks[name] = time.perf_counter()

    def n_in(self, a: str, b: str) -> int:
        ta, tb = self.marks.get(a, 0.0), self.marks.get(b, float("inf"))
        return sum(1 for t, _ in self.lines if ta <= t <= tb)

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self, min_samples: int = 3):
        window = "timed"
        sel = [ln for t, ln in self.lines if self.marks.get("start", 0) <= t <= self.marks.get("stop", 1e300)]
        if len(sel) < min_samples:
            window = "load (warm-up + timed + untimed tail of the same solves; timed region too short)"
            sel = [ln for t, ln in self.lines if self.marks.get("load", 0) <= t <= self.marks.get("end", 1e300)]
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in sel:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm), "window": window,
                "period_ms": self.PERIOD_MS}


# ---------------------------------------------------------------------------
# algorithmic bytes of the fused phase kernels


def phase_bytes(level, phase, fine: bool, c_only: bool = False) -> int:
    """Minimal HBM bytes one launch of a fused phase kernel must move.

    8 B per node for every state row read/written, every departure record
    (s) and sigma row read; GMRES Krylov traffic (on-chip/L2) is excluded."""
    from paper_2203_13382_b200 import _lib
    n = level.grid.n_points
    N = level.n_steps
    m = level.cf
    nI = N // m
    g = 0 if fine else 1           # G rows read (zero forcing on the fine level)
    d = level.grid.dim             # departure record and sigma: one fp64 per node per axis
    sig = d if level.kind != "fine" and level.sig_x is not None else 0
    # departure records: 8 B per node and axis, or one x-record per column and
    # one y-record per row (noise) on a separable plain-SL 2D level
    rec = 0 if (d == 2 and level.separable and level.kind in ("fine", "rediscretized")) else d
    # 2D steps are one batched launch per F-point offset: each step's input row
    # was written a whole batch (GBs) earlier and is read back from HBM; the 1D
    # phase kernels carry the row through an interval on chip
    inp = 1 if d == 2 else 0
    step = 8 * n * (rec + g + sig + inp + 1)   # s + G + sigma [+ input row] + output row
    if phase == _lib.PHASE_FC:
        left = 0 if (not fine or inp) else 8 * n
        if c_only:   # the fine FC phase runs only its C-step (mgrit._FusedCycle.skip_f)
            return nI * (step + (0 if inp else 8 * n))   # 1D: the last F row is read back
        return nI * (left + m * step)
    if phase == _lib.PHASE_F_RES:
        per = 8 * n * 2 + (m - 1) * step + 8 * n * (d + g + sig) + 8 * n * 3   # tail: s,G,sig + Cbuf r, U w, Gc w
        return nI * per
    if phase == _lib.PHASE_INJ_F:
        per = 8 * n * 3 + (m - 1) * step + (8 * n * (d + g + sig) + 16 * n if fine else 0)
        return nI * per
    return 0


def run_gpu(args):
    import torch
    import paper_2203_13382_b200 as P
    from paper_2203_13382_b200 import mgrit as M

    rank, world, local = _dist_env()
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        # eager communicator setup: every rank takes part in the first
        # collective (the engine's first op may be a one-sided P2P batch)
        dist.barrier()
    kw = dict(CONFIGS[args.config], gmres_variant=args.gmres_variant)
    P.set_launch_policy(args.launch_policy)
    cfg = P.SolverConfig(**kw)
    from paper_2203_13382_b200 import timepar as T
    comm = T.Comm() if world > 1 else None
    t0 = time.perf_counter()
    build_sharded = getattr(T, "build_hierarchy_sharded", None)
    levels = P.build_hierarchy(cfg) if world == 1 or build_sharded is None else build_sharded(cfg, comm)
    torch.cuda.synchronize()
    setup_s = time.perf_counter() - t0
    n_dof = cfg.n_x ** cfg.dim * cfg.n_t
    scfg = static_config(args.config)

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    def do_solve(iterate0=None, out=None):
        if world == 1:
            if iterate0 is None:
                return P.solve(cfg, levels, output="device")[0]
            return P.solve(cfg, levels, initial_iterate=iterate0, out=out)[0]
        return T.solve_time_parallel(cfg, levels, comm, iterate0=iterate0, out=out)[0]

    # inputs read by one solve: U plus the fine departure records (one shared
    # set for a constant speed).  Below twice the 126 MB L2 each timed solve
    # is preceded by an untimed write of a 256 MiB buffer, so no solve starts
    # with the previous one's data in L2.
    npts = cfg.n_x ** cfg.dim
    in_bytes = 8 * (cfg.n_t + 1) * npts + 8 * cfg.dim * npts * (1 if levels[0].shared else cfg.n_t)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda") if in_bytes < 2 * L2_BYTES else None

    # warm-up (also captures the CUDA graphs / sets kernel attributes)
    rep = do_solve()
    barrier()
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        clk.mark("load")
        for _ in range(args.warmup - 1):
            rep = do_solve()
        barrier()
        clk.mark("start")
        if flush is None:
            start.record()
            for _ in range(args.steps):
                rep = do_solve()
            stop.record()
            barrier()
            ms = start.elapsed_time(stop) / args.steps
        else:
            evs = []
            for _ in range(args.steps):
                flush.fill_(1)
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                rep = do_solve()
                b.record()
                evs.append((a, b))
            barrier()
            ms = sum(a.elapsed_time(b) for a, b in evs) / args.steps
        clk.mark("stop")
        if dist is not None:
            t = torch.tensor([ms], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        # untimed tail of the same solves so a very short timed region still
        # has clock samples taken under this load (reported as such); the
        # count derives from the all-reduced time, so every rank agrees
        if ms * args.steps < 3 * ClockSampler.PERIOD_MS + 60:
            for _ in range(min(int(300.0 / max(ms, 1e-3)) + 1, 2000)):
                do_solve()
            barrier()
        clk.mark("end")
    # the time-sharded solve does the whole problem once across all ranks
    # (strong scaling); replicas are not used
    value = n_dof / (ms / 1e3)

    # kernels launched per timed solve: the eager prologue (PCG64 fill, the
    # initial residual's row kernel(s), its fixed-order sum, the loop init)
    # plus, per iteration, the kernel nodes of the captured V-cycle + stop test
    if world == 1:
        sess = M._session(levels, cfg, torch.device("cuda"))
        body = sess.loop.body_kernels if sess.loop is not None else None
        eager = 4 + (1 if cfg.dim == 2 else 0)
        launches = eager + body * rep.iterations if body is not None and body >= 0 else None
    else:
        launches = getattr(T, "last_solve_launches", lambda: None)()

    # ---- end to end through the public API with host buffers: this rank's
    #      initial-iterate rows from pinned memory in, its U rows out
    row0, nrows = T.local_rows(cfg, levels, comm) if world > 1 else (0, cfg.n_t + 1)
    first = max(row0, 1)
    if args.no_e2e:
        Xp = Uh = torch.empty(0, dtype=torch.float64)
    else:
        # this rank's rows of numpy's default_rng(seed).random((n_t, n)),
        # drawn straight into pinned memory
        rng = np.random.default_rng(cfg.seed)
        if first > 1:
            rng.bit_generator.advance((first - 1) * npts)
        Xp = torch.empty((row0 + nrows - first, npts), dtype=torch.float64).pin_memory()
        rng.random(out=Xp.numpy())
        if cfg.iterate == "pm1":
            Xp.mul_(2.0).sub_(1.0)
        Uh = torch.empty((nrows, npts), dtype=torch.float64).pin_memory()
    e2e_ms = []
    for i in range(0 if args.no_e2e else max(2, min(args.steps, 4))):
        barrier()
        t1 = time.perf_counter()
        do_solve(iterate0=Xp, out=Uh)
        torch.cuda.synchronize()
        e2e_ms.append((time.perf_counter() - t1) * 1e3)
    e2e = float(np.median(e2e_ms[1:])) if e2e_ms else float("nan")
    if dist is not None:
        t = torch.tensor([e2e], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e = float(t.item())
    h2d, d2h = int(Xp.numel() * 8 + npts * 8) * world, int(Uh.numel() * 8) * world
    del Xp, Uh

    if rank != 0:
        if dist is not None:
            dist.barrier()
            dist.destroy_process_group()
        return
    clk_summary = clk.summary()
    roofline = sl_roof = breakdown = None
    seq = seq_forms = None
    if world == 1:
        # ---- per-launch breakdown of the first V-cycle (CUDA graphs, events)
        breakdown = kernel_breakdown(levels, cfg)
        roofline, sl_roof = _rooflines(args, cfg, levels, breakdown, clk_summary)
        seq, seq_forms = sequential_gpu(levels, cfg)
    parity = bench_parity(args.config, rep, P)
    iters = rep.iterations
    cpu = None
    if world == 1 and not args.no_cpu:
        cpu = cpu_baseline(args.config, iters, args.cpu_samples)
    line = {
        "metric": METRIC,
        "value": value, "unit": "DOF/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (BASELINE config; seeded PCG64 initial iterate, generated on the device)",
        "config": scfg,
        "solve": {"iterations": iters, "status": rep.status, "setup_s": round(setup_s, 4),
                  "final_factor": rep.final_factor, "gmres_variant": cfg.gmres_variant,
                  "launch_policy": args.launch_policy,
                  "parallelism": (f"time axis sharded over {world} GPUs (NCCL P2P halo rows, all-gathered "
                                  f"norm partials)") if world > 1 else "1 GPU"},
        "roofline": roofline,
        "sl_step_roofline": sl_roof,
        "cpu_baseline": cpu,
        "e2e": {"value": n_dof / (e2e / 1e3), "unit": "DOF/s", "ms_per_step": e2e,
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "path": "P.solve(cfg, levels, initial_iterate=<pinned host rows>, out=<pinned host U>)"},
        "clocks": clk_summary,
        "gpu_launches": launches,
        "parity": parity,
    }
    if seq is not None:
        line["sequential_gpu_ms"] = round(seq, 3)
        line["sequential_gpu_forms_ms"] = seq_forms
        line["speedup_vs_sequential_gpu"] = round(seq / ms, 4)
    if breakdown is not None:
        line["kernel_breakdown_ms"] = {k: round(v["ms_avg"] * v["launches"], 4) for k, v in breakdown.items()}
    if world > 1:
        line["nccl"] = {"backend": dist.get_backend(), "world_size": dist.get_world_size(),
                        "nccl_version": ".".join(map(str, torch.cuda.nccl.version()))}
    print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


def sequential_gpu(levels, cfg):
    """Plain sequential time stepping of the fine level (the sweep behind
    P.sequential_reference).  1D: the faster of the one-CTA sweep and the
    cluster-split sweep (the row split over up to 16 SMs, DSMEM/TMA-multicast
    row publication); returns (best ms, {form: ms})."""
    import paper_2203_13382_b200 as P
    if cfg.dim == 2:
        ms = _sequential_gpu_once(levels, cfg)
        return ms, {"batched_sl_steps": round(ms, 3)}
    forms = {}
    prev = P.set_launch_policy("cta")
    try:
        forms["one_cta"] = round(_sequential_gpu_once(levels, cfg), 3)
        P.set_launch_policy("cluster")
        try:
            forms["cluster"] = round(_sequential_gpu_once(levels, cfg), 3)
        except RuntimeError:
            pass   # row length not splittable over a cluster
    finally:
        P.set_launch_policy(prev)
    return min(forms.values()), forms


def _sequential_gpu_once(levels, cfg) -> float:
    """One form of the sweep; state buffer and u0 prepared outside the timing."""
    import torch
    from paper_2203_13382_b200 import mgrit as M
    npts = cfg.n_x ** cfg.dim
    Useq = torch.empty((cfg.n_t + 1, npts), dtype=torch.float64, device="cuda")
    Useq[0] = torch.from_numpy(M.initial_state(cfg, levels[0].grid)).cuda()
    for _ in range(2):
        M._sweep(levels[0], Useq, None, zero_init=False)
    torch.cuda.synchronize()
    # 2D steps are one launch each: replay them from a CUDA graph, so the
    # baseline carries no host launch overhead (1D: one persistent kernel)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        M._sweep(levels[0], Useq, None, zero_init=False)
    g.replay()
    torch.cuda.synchronize()
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0.record()
    for _ in range(3):
        g.replay()
    s1.record()
    torch.cuda.synchronize()
    return s0.elapsed_time(s1) / 3


def _rooflines(args, cfg, levels, breakdown, clk_summary):
    top = max(breakdown, key=lambda k: breakdown[k]["ms_avg"] * breakdown[k]["launches"])
    tb = breakdown[top]
    peak = _peak()
    achieved = tb["bytes"] / (tb["ms_avg"] / 1e3) / 1e9
    if "corrected" not in top:
        limiter = ("instruction issue of the separable SL step (DESIGN.md section 4)" if cfg.dim == 2 and levels[0].separable
                   else "FP64 issue + L1 gather wavefronts (DESIGN.md section 4)")
    elif cfg.dim == 1:
        limiter = "latency: MGS-GMRES reduction chain of a few row chains (see DESIGN.md section 4)"
    else:
        limiter = ("Krylov passes of the cooperative GMRES through L2/HBM with two systems in flight, ~17 dependent "
                   "pass + barrier intervals per system (DESIGN.md section 4, profiles/r02g_probe_coop2d_cfg5mesh_k4.txt)")
    total = sum(v["ms_avg"] * v["launches"] for v in breakdown.values())
    roofline = {"bound": "hbm", "limiter": limiter, "kernel": top, "achieved": round(achieved, 1),
                "peak": peak["hbm_gbs"], "unit": "GB/s", "frac": round(achieved / peak["hbm_gbs"], 4),
                "traffic": _ncu_traffic(args.config, top), "bytes_per_launch": tb["bytes"],
                "ms_per_launch": round(tb["ms_avg"], 5), "peak_source": peak["source"],
                "share_of_iteration": round(tb["ms_avg"] * tb["launches"] / total, 3),
                "timing": "CUDA events on the launching stream around a graph replay of the phase, "
                          "state restored to the first V-cycle's before each replay"}
    ops = _ncu_fp64(cfg.dim, cfg.p, cfg.dim == 2 and bool(levels[0].separable))
    sm_mhz = clk_summary.get("sm_mhz") or 1965.0
    fpeak = 148 * 64 * sm_mhz * 1e6 / 1e12
    if "corrected" not in top and ops:
        lv0 = levels[0]
        steps_top = lv0.n_steps // lv0.cf if tb.get("c_only") else lv0.n_steps
        fach = ops * steps_top * lv0.grid.n_points / (tb["ms_avg"] / 1e3) / 1e12
        roofline["fp64"] = {"achieved": round(fach, 2), "peak": round(fpeak, 2), "unit": "T FP64 inst/s",
                            "frac": round(fach / fpeak, 4), "ops_per_node_update": ops}
    if "corrected" in top and cfg.dim == 1 and "sweep" not in top:
        li = int(top[1:].split("_")[0])
        m = levels[li].cf
        steps = m - 1 if "INJ_F" in top else m
        us_step = tb["ms_avg"] * 1e3 / steps
        roofline["latency"] = {
            "row_chains": levels[li].n_steps // m, "steps_per_chain": steps,
            "us_per_corrected_step": round(us_step, 2),
            "cycles_per_corrected_step_at_1965MHz": int(us_step * 1965),
            "note": "each corrected step is an SL gather + MGS-GMRES with up to 10 Arnoldi steps; "
                    "every MGS projection is one cluster all-reduce, so the step is bound by ~K^2/2 "
                    "dependent all-reduces, not by bytes"}

    # the SL-step kernel itself (BASELINE: "SL-step HBM GB/s"): the fine-level
    # F+C relaxation phase (plain semi-Lagrangian steps, G = 0)
    # 2D: the FC phase (since round 2 exactly one batched SL step of every
    # interval); 1D: the fused F-relaxation + C-point residual phase (the FC
    # phase is a small C-step-only row launch there)
    pref = ("L0_FC", "L0_FONLY") if cfg.dim == 2 else ("L0_F_RES", "L0_FONLY", "L0_FC")
    sl_key = next((k for pfx in pref for k in breakdown if k.startswith(pfx)), None)
    sl_roof = None
    if sl_key is not None:
        sb = breakdown[sl_key]
        ach = sb["bytes"] / (sb["ms_avg"] / 1e3) / 1e9
        hbm_frac = ach / peak["hbm_gbs"]
        sl_roof = {"bound": "hbm", "kernel": sl_key, "achieved": round(ach, 1), "peak": peak["hbm_gbs"],
                   "unit": "GB/s", "frac": round(hbm_frac, 4), "traffic": _ncu_traffic(args.config, sl_key),
                   "bytes_per_launch": sb["bytes"], "ms_per_launch": round(sb["ms_avg"], 5),
                   "note": ("plain SL steps of the fine level on separable records: 8 B input row + 8 B new row "
                            "per node-update (one x-record per column and one y-record per row)")
                   if (cfg.dim == 2 and levels[0].separable) else
                   "plain SL steps of the fine level (8 B record per axis + 8 B new row per node-update"
                   + (" + 8 B input row)" if cfg.dim == 2 else ")")}
        if ops:
            lv0 = levels[0]
            node_updates = (lv0.n_steps // lv0.cf if (sb.get("c_only") and sl_key.startswith("L0_FC"))
                            else lv0.n_steps) * lv0.grid.n_points
            fach = ops * node_updates / (sb["ms_avg"] / 1e3) / 1e12
            sl_roof["fp64"] = {"achieved": round(fach, 2), "peak": round(fpeak, 2), "unit": "T FP64 inst/s",
                               "frac": round(fach / fpeak, 4), "ops_per_node_update": ops,
                               "source": "profiles/ncu_fp64.json (ncu SASS counts)"}
            sl_roof["binding"] = "fp64" if fach / fpeak > hbm_frac else "hbm"
    return roofline, sl_roof


def kernel_breakdown(levels, cfg, reps: int = 3):
    """Device time of every launch of the solve's FIRST V-cycle.  Walking the
    cycle in order, each phase launch is captured into its own CUDA graph;
    the engine state (every level's U/G/C buffers) is snapshotted before the
    phase and restored before each replay, so every timed replay sees exactly
    the first V-cycle's data (a corrected step's GMRES stops on breakdown or
    tolerance, so its cost depends on the data) and the walk continues from
    the state one application produces."""
    import torch
    from paper_2203_13382_b200 import _lib
    from paper_2203_13382_b200 import mgrit as M
    dev = torch.device("cuda")
    eng = M._session(levels, cfg, dev).engine
    U = eng.U[0]
    U[0] = M._initial_row(cfg, levels[0], dev)
    M.pcg64_uniform(cfg.seed, cfg.n_t, levels[0].grid.n_points, U[1:], pm1=(cfg.iterate == "pm1"))
    eng.prologue()   # as solve() does: 2D fine F-points relaxed once, before the first V-cycle
    state = [t for t in list(eng.U) + list(eng.G) + list(eng.C) + [eng.partial] if t is not None]
    torch.cuda.synchronize()
    names = {_lib.PHASE_FC: "FC", _lib.PHASE_F_RES: "F_RES", _lib.PHASE_FONLY_RES: "FONLY_RES",
             _lib.PHASE_INJ_F: "INJ_F"}
    order = []

    def walk(li=0):
        if li == len(levels) - 1:
            order.append((f"L{li}_sweep_{levels[li].kind}", lambda li=li: eng.cycle(li), 0))
            return
        seq = [_lib.PHASE_FC, _lib.PHASE_F_RES] if eng.relaxation == "FCF" else [_lib.PHASE_FONLY_RES]
        for ph in seq:
            order.append((f"L{li}_{names[ph]}_{levels[li].kind}", lambda li=li, ph=ph: eng._phase(li, ph),
                          phase_bytes(levels[li], ph, li == 0,
                                      c_only=(li == 0 and ph == _lib.PHASE_FC and eng.skip_f))))
        walk(li + 1)
        ph = _lib.PHASE_INJ_F
        order.append((f"L{li}_{names[ph]}_{levels[li].kind}", lambda li=li, ph=ph: eng._phase(li, ph),
                      phase_bytes(levels[li], ph, li == 0)))

    walk()
    out = {}
    stream = torch.cuda.current_stream()
    for key, fn, nbytes in order:
        snap = [t.clone() for t in state]
        fn()                              # kernel attributes, first-use setup (undone by the restore)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            fn()
        ts = []
        for r in range(reps + 1):
            for t, s in zip(state, snap):
                t.copy_(s)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            g.replay()
            b.record(stream)
            torch.cuda.synchronize()
            if r:
                ts.append(a.elapsed_time(b))
        del snap, g
        ms = float(np.median(ts))
        o = out.setdefault(key, {"ms_avg": ms, "bytes": nbytes, "launches": 0,
                                 "c_only": bool(key.startswith("L0_FC") and eng.skip_f)})
        o["launches"] += 1
    return out


def bench_parity(name, rep, P):
    """Iteration count / status / residual history of the timed solve against
    the full-size reference history where one exists."""
    hist = np.asarray(rep.residual_norms)
    g = GOLDEN.get(name)
    if g is not None:
        with open(os.path.join(ROOT, "tests", "golden", "index.json")) as f:
            info = json.load(f).get(g)
        if info is None:
            return None
        ref = np.load(os.path.join(ROOT, "tests", "golden", f"solve_{g}.npz"))["hist"]
        dev = float(np.max(np.abs(hist - ref)) / ref[0]) if len(ref) == len(hist) else None
        return {"fixture": f"tests/golden/solve_{g}.npz", "source": "reference mgrit_advect, full size",
                "iterations": rep.iterations, "reference_iterations": info["iterations"],
                "status": rep.status, "reference_status": info["status"], "max_history_dev_over_r0": dev}
    fx = FULLSIZE.get(name)
    if fx is not None:
        return _fixture_parity(fx, hist, rep)
    if name == "cfg5":
        return _cfg5_mesh_parity(P)
    return None


def _load_fixture(fx):
    path = os.path.join(ROOT, "tests", "golden", f"solve_{fx}.npz")
    if not os.path.exists(path):
        return None
    g = dict(np.load(path))
    g["meta"] = json.loads(str(g["meta"]))
    return g


def _fixture_parity(fx, hist, rep):
    g = _load_fixture(fx)
    if g is None:
        return {"fixture": None, "note": f"tests/golden/solve_{fx}.npz not generated"}
    meta = g["meta"]
    ref = g["hist"]
    k = min(len(ref), len(hist))
    out = {"fixture": f"tests/golden/solve_{fx}.npz", "source": meta["source"],
           "reference_status": meta["status"], "reference_iterations_recorded": meta["iterations"],
           "iterations": rep.iterations, "status": rep.status,
           "compared_iterations": k - 1,
           "max_history_dev_over_r0": float(np.max(np.abs(hist[:k] - ref[:k])) / ref[0])}
    if meta["status"] == "converged":
        out["iterations_equal"] = bool(meta["iterations"] == rep.iterations)
    return out


def _cfg5_mesh_parity(P):
    """Config 5 itself has no CPU reference; its mesh,
    degree, factor, speed, seed and u0 on 128 steps do (real reference,
    2 V-cycles): solve that here with the same kernels and compare."""
    g = _load_fixture(CFG5_MESH_FIXTURE)
    if g is None:
        return {"fixture": None, "note": "no full-size CPU reference for cfg5"}
    meta = g["meta"]
    k = meta["iterations"]
    cfg = P.SolverConfig(**{**meta["kw"], "max_iters": k, "rtol": 0.0})
    rep, U = P.solve(cfg)
    ref = g["hist"]
    rows = float(np.max(np.abs(np.linalg.norm(U, axis=1) - g["row_norms"][k - 1]) / g["row_norms"][k - 1]))
    return {"fixture": f"tests/golden/solve_{CFG5_MESH_FIXTURE}.npz", "source": meta["source"],
            "workload": "cfg5's 1024^2 mesh, p=5, m=8, speed, seed 4 and u0 on 128 of the 2048 steps "
                        "(levels [128, 16, 2]); the full cfg5 needs > 150 GB and hours per V-cycle on the CPU",
            "compared_iterations": k, "max_history_dev_over_r0": float(np.max(np.abs(rep.residual_norms - ref)) / ref[0]),
            "max_row_norm_rel_dev": rows}


def _peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return {"hbm_gbs": float(d["hbm_gbs"]), "source": "measured (MEASURED_PEAKS.json)"}
    return {"hbm_gbs": 6650.0, "source": "fallback (B200_PROFILING.md)"}


def _ncu_fp64(dim, p, separable=False):
    """FP64 instructions per node-update of the fine SL kernel (ncu-measured)."""
    path = os.path.join(ROOT, "profiles", "ncu_fp64.json")
    if not os.path.exists(path):
        return None
    with open(path) as f:
        d = json.load(f)
    return d.get(f"{dim}d_p{p}_sep" if separable else f"{dim}d_p{p}", d.get(f"{dim}d_p{p}"))


def _ncu_traffic(config, kernel_key):
    """DRAM bytes per launch from the committed ncu --set full summary, if any."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(p):
        return None
    with open(p) as f:
        d = json.load(f)
    return d.get(f"{config}:{kernel_key}")


# ---------------------------------------------------------------------------
# CPU legs (oracle = the reference's algorithm, bit-identical)


_ORACLE = {}


def _vcycle_sample(name: str):
    """cfg1/cfg2: one V-cycle + convergence residual on the host (seconds),
    plus the initial-residual time (hierarchy built once, outside the sample)."""
    import oracle as O
    ocfg = O.OConfig(**CONFIGS[name])
    if name not in _ORACLE:
        _ORACLE[name] = O.hierarchy(ocfg)
    levels = _ORACLE[name]
    fine = levels[0]
    U = np.empty((ocfg.n_t + 1, fine.n_points))
    U[0] = O.initial_state(ocfg)
    U[1:] = O.initial_iterate(ocfg)
    G = np.zeros_like(U)
    t0 = time.perf_counter()
    O.st_norm(O.residual(fine, U, G))
    t_r0 = time.perf_counter() - t0
    t1 = time.perf_counter()
    O.v_cycle(levels, 0, U, G, ocfg.relaxation)
    O.st_norm(O.residual(fine, U, G))
    return t_r0, time.perf_counter() - t1


def _model_levels(name: str):
    """Full-size oracle operators for the per-application model: the fine
    level's step 0 (ERK departures) and the first coarse level's step 0
    (backtracked through its m fine children, sigma from phi)."""
    import oracle as O
    if name in _ORACLE:
        return _ORACLE[name]
    kw = CONFIGS[name]
    ocfg = O.OConfig(**kw)
    dim, nx, p = ocfg.dim, ocfg.n_x, ocfg.p
    dt = ocfg.dt if ocfg.dt is not None else 0.85 * 2.0 / nx
    sizes, factors = level_sizes(kw)
    m = factors[0]
    t0 = time.perf_counter()
    shared = O.speed_is_constant(ocfg.wave_speed)
    children = [O.erk_departures(dim, nx, ocfg.wave_speed, k * dt, dt, ocfg.order) for k in range(1 if shared else m)]
    if shared:
        children = children * m
    fine = O.OLevel(0, dim, nx, p, sizes[0], dt, "fine", children[:1])
    coarse_dep = O.backtrack(dim, nx, children)
    sig = O.phi_sigma(p, coarse_dep, children, None)
    gm = (10, None) if len(sizes) == 2 else (10, 1e-2)
    coarse = O.OLevel(1, dim, nx, p, sizes[1], dt * m, "corrected", [coarse_dep], [sig], gmres=gm)
    u = np.random.default_rng(ocfg.seed).random(nx ** dim)
    _ORACLE[name] = (fine, coarse, u, sizes, factors, time.perf_counter() - t0)
    return _ORACLE[name]


def _model_sample(name: str):
    """One full-size fine SL step and one full-size corrected coarse step
    (the random initial-iterate row as input), seconds; + its Arnoldi count."""
    import oracle as O
    fine, coarse, u, *_ = _model_levels(name)
    t0 = time.perf_counter()
    fine.step(0, u)
    t_sl = time.perf_counter() - t0
    log = O.GmresLog()
    coarse.log = log
    t1 = time.perf_counter()
    coarse.step(0, u)
    return t_sl, time.perf_counter() - t1, log.counts[-1]


def applications(name: str):
    """Operator applications of one reference solve iteration (mgrit.py:276-334
    plus the convergence residual, mgrit.py:368): per non-coarsest level N steps
    of F-relax (N(m-1)/m) x 3, C-relax (N/m) and the residual (N) -> N(4 - 2/m);
    the coarsest level N; the fine level adds the convergence residual N."""
    sizes, factors = level_sizes(CONFIGS[name])
    per = []
    for li, (N, m) in enumerate(zip(sizes, factors)):
        a = N * (4.0 - 2.0 / m) if m else float(N)
        if li == 0:
            a += N
        per.append(a)
    return per


def model_estimate(name: str, t_sl: float, t_corr: float, iters: int):
    per = applications(name)
    t_iter = per[0] * t_sl + sum(per[1:]) * t_corr
    return CONFIGS[name]["n_t"] * t_sl + iters * t_iter, t_iter


def cpu_sample(name: str, iters: int):
    """(estimated full-solve seconds, description) from one bounded sample."""
    if name in GOLDEN:
        t_r0, t_it = _vcycle_sample(name)
        return t_r0 + iters * t_it, (f"one V-cycle with convergence residual ({t_it:.2f} s) + initial residual "
                                     f"({t_r0:.2f} s) of {name}, extrapolated x{iters} iterations")
    t_sl, t_corr, k = _model_sample(name)
    est, t_iter = model_estimate(name, t_sl, t_corr, iters)
    per = applications(name)
    return est, (f"extrapolated: one full-size fine SL step ({t_sl:.3f} s) and one full-size corrected "
                 f"coarse step ({t_corr:.3f} s, {k} Arnoldi steps) timed; x {int(per[0])} fine and "
                 f"{int(sum(per[1:]))} coarse applications per iteration (mgrit.py:276-334) = "
                 f"{t_iter:.0f} s/iteration, x{iters} iterations + initial residual")


def _iters_for(name: str) -> tuple[int, str]:
    g = GOLDEN.get(name)
    if g is not None:
        with open(os.path.join(ROOT, "tests", "golden", "index.json")) as f:
            return json.load(f)[g]["iterations"], "the reference's own full-size solve"
    fx = FULLSIZE.get(name)
    if fx is not None:
        fix = _load_fixture(fx)
        if fix is not None and fix["meta"]["status"] == "converged":
            return fix["meta"]["iterations"], f"full-size fixture tests/golden/solve_{fx}.npz ({fix['meta']['source']})"
    return EXTRAP_ITERS[name]


def cpu_baseline(name: str, iters: int, samples: int = 1):
    n_dof = CONFIGS[name]["n_x"] ** CONFIGS[name].get("dim", 1) * CONFIGS[name]["n_t"]
    best = None
    for _ in range(max(1, samples)):
        est, desc = cpu_sample(name, iters)
        best = (est, desc) if best is None or est < best[0] else best
    return {"value": n_dof / best[0], "unit": "DOF/s", "cores": 1, "kind": "port",
            "sample": f"oracle (bit-identical numpy/C restatement of mgrit_advect): {best[1]}; setup excluded",
            "host_cpus": os.cpu_count(),
            "cores_note": "the reference runs single-threaded numpy / numba (its corrected levels loop over "
                          "rows in Python, Level.step_batch mgrit.py:152-167); one core is what it uses"}


def run_reference(args):
    rank, world, _ = _dist_env()
    if rank != 0:
        return
    name = args.config
    iters, iters_src = _iters_for(name)
    n_dof = CONFIGS[name]["n_x"] ** CONFIGS[name].get("dim", 1) * CONFIGS[name]["n_t"]
    times, desc = [], ""
    for i in range(args.warmup + args.steps):
        est, desc = cpu_sample(name, iters)
        if i >= args.warmup:
            times.append(est)
    est = float(np.mean(times))
    value = n_dof / est
    line = {
        "impl": "reference", "metric": METRIC, "value": value,
        "unit": "DOF/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": est * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (BASELINE config; seeded PCG64 initial iterate)",
        "config": static_config(name),
        "cpu_baseline": {"value": value, "unit": "DOF/s", "cores": 1, "kind": "port",
                         "sample": f"per step: {desc}; iterations from {iters_src}; setup excluded",
                         "host_cpus": os.cpu_count()},
        "e2e": {"value": value, "unit": "DOF/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "extrapolated": True,
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# launcher


def _free_port() -> int:
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def spawn(n: int, argv: list[str]) -> int:
    """Re-launch this script under torch.distributed.run with n ranks (one GPU
    each; rendezvous on 127.0.0.1).  NCCL's INIT log goes to stderr so the
    communicators (nRanks) are visible without touching the JSON line."""
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    env.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__), *argv]
    return subprocess.call(cmd, env=env)


def launch_check(args):
    """Launcher self-test (CPU, gloo): every rank reports in; rank 0 prints."""
    import torch
    import torch.distributed as dist
    rank, world, local = _dist_env()
    dist.init_process_group("gloo")
    got = [None] * world
    dist.all_gather_object(got, {"rank": rank, "local_rank": local, "world": world, "pid": os.getpid()})
    if rank == 0:
        print(json.dumps({"launch_check": True, "n_gpus": args.gpus, "world_size": world, "ranks": got}),
              flush=True)
    dist.barrier()
    dist.destroy_process_group()
    del torch


def main(argv=None):
    argv = sys.argv[1:] if argv is None else argv
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default=DEFAULT_CONFIG, choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--cpu-samples", type=int, default=1)
    ap.add_argument("--gmres-variant", default="mgs", choices=["mgs", "mgs_lowsync"],
                    help="coarse-level Arnoldi orthogonalisation (mgs = the reference's loop)")
    ap.add_argument("--launch-policy", default="auto", choices=["auto", "cta", "cluster", "auto_one"],
                    help="corrected 1D kernels: one CTA or one 8-SM cluster per row chain")
    ap.add_argument("--no-e2e", action="store_true", help="skip the host-buffer end-to-end leg")
    ap.add_argument("--launch-check", action="store_true", help=argparse.SUPPRESS)
    args = ap.parse_args(argv)
    if args.warmup < 3:
        args.warmup = 3
    if "WORLD_SIZE" not in os.environ:
        if args.gpus > 1:
            return spawn(args.gpus, argv)
    elif int(os.environ["WORLD_SIZE"]) != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={os.environ['WORLD_SIZE']}")
    if args.launch_check:
        launch_check(args)
    elif args.impl == "reference":
        run_reference(args)
    else:
        run_gpu(args)
    return 0


if __name__ == "__main__":
    sys.exit(main())
