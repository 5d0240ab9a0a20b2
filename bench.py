"""Benchmark: MGRIT solve space-time DOF/s to 1e-10 relative residual.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg2] [--impl reference]

One *step* = one complete MGRIT solve (BASELINE.json metric) of the chosen
config from the prebuilt device hierarchy: U initialisation (numpy PCG64
stream generated bit-identically on the device), initial residual, V-cycles
and convergence residuals until ||r|| <= 1e-10 ||r0||.  Hierarchy setup
(ERK tracing, backtracking, sigma) is excluded and reported separately, as in
the reference's timing discussion.

Default workload: BASELINE config 2 (configs[1]): 1D, n_x = n_t = 4096,
a(x,t) = 1 + 0.5 sin(2 pi x) cos(2 pi t), p = 3, m = 4, FCF, multilevel
(6 levels), seed 1, dt = 0.85 h (reference default).  U (134 MB) and the
fine departure records (134 MB) exceed the 126 MB L2, so no explicit flush;
workloads under twice the L2 (cfg1) get an untimed 256 MiB write before each
timed solve instead.

``--impl reference`` times the reference's CPU implementation of the path —
the oracle port under oracle/ (bit-identical to mgrit_advect; the reference
is pure Python so there is nothing to compile into oracle/_ref) — on the
host cores, one bounded sample (one V-cycle + convergence residual of the
same config) per step, extrapolated to a full solve with the reference's own
iteration count.

N > 1 (torchrun): the time axis of the one solve is sharded across the ranks
(paper_2203_13382_b200/timepar.py; NCCL send/recv of boundary C-point rows,
all-gathered norm partials) — "scaling": "strong" (fixed total work).
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
DESCR = {
    "cfg1": "BASELINE cfg1: 1D a=1, 1024x1024, p=1, two-level m=8, dt=2/nt (CFL 1), iterate U[-1,1) seed 0",
    "cfg1_085h": "BASELINE cfg1 mesh at dt=0.85h (non-degenerate companion)",
    "cfg2": "BASELINE cfg2: 1D a=1+0.5sin(2pi x)cos(2pi t), 4096x4096, p=3, m=4 multilevel FCF, seed 1, dt=0.85h",
    "cfg3": "BASELINE cfg3: 1D same speed, 16384x16384, p=5, m=8 multilevel FCF, seed 2, dt=0.85h",
    "cfg4": "BASELINE cfg4: 2D a=(cos^2(pi x)cos(2pi t)+.5, sin^2(pi y)cos(2pi t)+.5), 512^2 x 1024, p=3, m=4, "
            "u0=sin^4 sin^4, seed 3, dt=0.85h",
    "cfg5": "BASELINE cfg5: 2D same speed, 1024^2 x 2048, p=5, m=8, u0=sin^4 sin^4, seed 4, dt=0.85h",
}
GOLDEN = {"cfg1": "cfg1_full", "cfg1_085h": "cfg1_085h", "cfg2": "cfg2_full"}


L2_BYTES = 126 * 1024 * 1024   # B200 L2

def _golden(name):
    g = GOLDEN.get(name)
    if g is None:
        return None
    with open(os.path.join(ROOT, "tests", "golden", "index.json")) as f:
        ix = json.load(f)
    if g not in ix:
        return None
    hist = np.load(os.path.join(ROOT, "tests", "golden", f"solve_{g}.npz"))["hist"]
    return ix[g], hist


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


def phase_bytes(level, phase, fine: bool) -> int:
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
    step = 8 * n * (d + g + sig + 1)   # s + G + sigma + output row
    if phase == _lib.PHASE_FC:
        left = 0 if not fine else 8 * n
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
    from paper_2203_13382_b200 import _lib
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
    t0 = time.perf_counter()
    levels = P.build_hierarchy(cfg)
    torch.cuda.synchronize()
    setup_s = time.perf_counter() - t0
    n_dof = cfg.n_x ** cfg.dim * cfg.n_t

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    from paper_2203_13382_b200 import timepar as T
    comm = T.Comm() if world > 1 else None

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
    npts_ = cfg.n_x ** cfg.dim
    in_bytes = 8 * (cfg.n_t + 1) * npts_ + 8 * cfg.dim * npts_ * (1 if levels[0].shared else cfg.n_t)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda") if in_bytes < 2 * L2_BYTES else None

    # warm-up (also compiles CUDA graphs / sets kernel attributes)
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

    # ---- end to end through the public API with host buffers: this rank's
    #      initial-iterate rows from pinned memory in, its U rows out
    npts = cfg.n_x ** cfg.dim
    row0, nrows = T.local_rows(cfg, levels, comm) if world > 1 else (0, cfg.n_t + 1)
    first = max(row0, 1)
    if args.no_e2e:
        Xp = Uh = torch.empty(0, dtype=torch.float64)
    else:
        X = torch.from_numpy(np.random.default_rng(cfg.seed).random((cfg.n_t, npts))[first - 1: row0 + nrows - 1])
        if cfg.iterate == "pm1":
            X = 2.0 * X - 1.0
        Xp = X.contiguous().pin_memory()
        Uh = torch.empty((nrows, npts), dtype=torch.float64).pin_memory()
    e2e_ms = []
    for i in range(0 if args.no_e2e else max(2, min(args.steps, 5))):
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

    if rank != 0:
        if dist is not None:
            dist.barrier()
            dist.destroy_process_group()
        return
    clk_summary = clk.summary()
    # ---- per-kernel breakdown of one single-GPU V-cycle (eager launches, CUDA events)
    breakdown, launches_iter = kernel_breakdown(levels, cfg)
    top = max(breakdown, key=lambda k: breakdown[k]["ms_total"])
    tb = breakdown[top]
    peak = _peak()
    achieved = tb["bytes"] / (tb["ms_avg"] / 1e3) / 1e9
    if "corrected" not in top:
        limiter = "FP64 issue + HBM"
    elif cfg.dim == 1:
        limiter = "latency: MGS-GMRES reduction chain of a few row chains (see DESIGN.md section 4)"
    else:
        limiter = "per-system barriers + L2-resident Krylov passes of the cooperative GMRES (DESIGN.md section 4)"
    roofline = {"bound": "hbm", "limiter": limiter, "kernel": top, "achieved": round(achieved, 1),
                "peak": peak["hbm_gbs"],
                "unit": "GB/s", "frac": round(achieved / peak["hbm_gbs"], 4),
                "traffic": _ncu_traffic(args.config, top), "bytes_per_launch": tb["bytes"],
                "ms_per_launch": round(tb["ms_avg"], 5), "peak_source": peak["source"],
                "share_of_iteration": round(tb["ms_total"] / sum(v["ms_total"] for v in breakdown.values()), 3)}
    if "corrected" in top and cfg.dim == 1 and "sweep" not in top:
        # the latency view of a corrected phase: when its row chains fit in
        # one wave, the launch time is steps-per-chain dependent corrected
        # steps (a level with more chains than resident CTAs / clusters runs
        # several waves, and the per-step figure is an upper bound)
        li = int(top[1:].split("_")[0])
        m = levels[li].cf
        steps = m - 1 if "INJ_F" in top else m
        us_step = tb["ms_avg"] * 1e3 / steps
        roofline["latency"] = {
            "row_chains": levels[li].n_steps // m, "steps_per_chain": steps,
            "us_per_corrected_step": round(us_step, 2),
            "cycles_per_corrected_step_at_1965MHz": int(us_step * 1965),
            "note": "each corrected step is an SL gather + MGS-GMRES with up to 10 Arnoldi steps; "
                    "every MGS projection is one cluster all-reduce (~580 cycles: fp64 warp butterfly "
                    "~200 + DSMEM round trip ~300, clock64 probe), so the step is bound by ~K^2/2 "
                    "dependent all-reduces, not by bytes"}

    # the SL-step kernel itself (BASELINE: "SL-step HBM GB/s"): the fine-level
    # F+C relaxation phase (plain semi-Lagrangian steps, G = 0)
    sl_key = next((k for k in breakdown if k.startswith("L0_FC") or k.startswith("L0_FONLY")), None)
    sl_roof = None
    if sl_key is not None:
        sb = breakdown[sl_key]
        ach = sb["bytes"] / (sb["ms_avg"] / 1e3) / 1e9
        hbm_frac = ach / peak["hbm_gbs"]
        sl_roof = {"bound": "hbm", "kernel": sl_key, "achieved": round(ach, 1), "peak": peak["hbm_gbs"],
                   "unit": "GB/s", "frac": round(hbm_frac, 4), "traffic": _ncu_traffic(args.config, sl_key),
                   "bytes_per_launch": sb["bytes"], "ms_per_launch": round(sb["ms_avg"], 5),
                   "note": "plain SL steps of the fine level (8 B record per axis + 8 B new row per node-update)"}
        # the same launch against the FP64 issue rate: ncu-counted FP64
        # instructions per node-update x node-updates / time
        ops = _ncu_fp64(cfg.dim, cfg.p)
        if ops:
            lv0 = levels[0]
            node_updates = lv0.n_steps * lv0.grid.n_points
            sm_mhz = clk_summary.get("sm_mhz") or 1965.0
            fpeak = 148 * 64 * sm_mhz * 1e6 / 1e12
            fach = ops * node_updates / (sb["ms_avg"] / 1e3) / 1e12
            sl_roof["fp64"] = {"achieved": round(fach, 2), "peak": round(fpeak, 2), "unit": "T FP64 inst/s",
                               "frac": round(fach / fpeak, 4), "ops_per_node_update": ops,
                               "source": "profiles/ncu_fp64.json (ncu SASS counts)"}
            sl_roof["binding"] = "fp64" if fach / fpeak > hbm_frac else "hbm"

    # ---- sequential GPU time stepping of the fine level (the sweep behind
    #      P.sequential_reference: 1D one CTA walks all steps, 2D one batched
    #      launch per step); state buffer and u0 prepared outside the timing
    Useq = torch.empty((cfg.n_t + 1, npts), dtype=torch.float64, device="cuda")
    Useq[0] = torch.from_numpy(M.initial_state(cfg, levels[0].grid)).cuda()
    for _ in range(2):
        M._sweep(levels[0], Useq, None, zero_init=False)
    torch.cuda.synchronize()
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0.record()
    for _ in range(3):
        M._sweep(levels[0], Useq, None, zero_init=False)
    s1.record()
    torch.cuda.synchronize()
    seq_ms = s0.elapsed_time(s1) / 3
    del Useq

    iters = rep.iterations
    # pcg fill + r0 (rows + sum) + loop init, then per iteration the V-cycle
    # launches, the norm sum and the device loop's stop test
    launches = 3 + 1 + (launches_iter + 1) * iters if world == 1 else 3 + launches_iter * iters
    parity = None
    gold = _golden(args.config)
    if gold is not None:
        info, hist = gold
        dev_r0 = float(np.max(np.abs(rep.residual_norms - hist)) / hist[0]) if len(hist) == len(rep.residual_norms) else None
        parity = {"iterations": iters, "reference_iterations": info["iterations"], "status": rep.status,
                  "max_history_dev_over_r0": dev_r0}
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline(args.config, iters, args.cpu_samples)
    if rank == 0:
        line = {
            "metric": "MGRIT solve space-time DOF/s to 1e-10 residual",
            "value": value, "unit": "DOF/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic (BASELINE config; seeded PCG64 initial iterate)",
            "config": {"workload": DESCR[args.config], "name": args.config, "n_x": cfg.n_x, "n_t": cfg.n_t,
                       "p": cfg.p, "schedule": cfg.schedule, "levels": [lv.n_steps for lv in levels],
                       "dt": levels[0].dt, "parallelism": f"time-sharded over {world} GPUs (NCCL halo rows)" if world > 1 else "1gpu",
                       "l2": (f"inputs larger than L2 ({in_bytes / 2**20:.0f} MiB of U + fine departure records "
                              f"> {L2_BYTES / 2**20:.0f} MiB)" if flush is None else
                              f"L2 flushed before every timed solve (untimed 256 MiB write; inputs "
                              f"{in_bytes / 2**20:.0f} MiB < 2 x {L2_BYTES / 2**20:.0f} MiB L2)"),
                       "setup_s": round(setup_s, 4), "iterations": iters, "status": rep.status,
                       "gmres_variant": cfg.gmres_variant, "launch_policy": args.launch_policy},
            "roofline": roofline,
            "sl_step_roofline": sl_roof,
            "cpu_baseline": cpu,
            "e2e": {"value": n_dof / (e2e / 1e3), "unit": "DOF/s", "ms_per_step": e2e,
                    "h2d_bytes_per_step": int(Xp.numel() * 8 + npts * 8) * world,
                    "d2h_bytes_per_step": int(Uh.numel() * 8) * world},
            "clocks": clk_summary,
            "gpu_launches": launches,
            "sequential_gpu_ms": round(seq_ms, 3),
            "speedup_vs_sequential_gpu": round(seq_ms / ms, 4),
            "kernel_breakdown_ms": {k: round(v["ms_total"], 4) for k, v in breakdown.items()},
            "parity": parity,
        }
        print(json.dumps(line))
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


def kernel_breakdown(levels, cfg, inner: int = 5, reps: int = 3):
    """Device time of every launch of one V-cycle: each launch (in cycle order)
    is captured `inner` times into its own CUDA graph and replayed between CUDA
    events on the launching stream, so host launch overhead is excluded.
    Repeating a phase is harmless for timing (the phases are idempotent except
    INJ_F, whose repeated injection only changes values)."""
    import torch
    from paper_2203_13382_b200 import _lib
    from paper_2203_13382_b200 import mgrit as M
    dev = torch.device("cuda")
    U = torch.empty((cfg.n_t + 1, levels[0].grid.n_points), dtype=torch.float64, device=dev)
    # the solve's own first iterate (u0 row + seeded PCG64 rows): corrected
    # steps stop GMRES early on breakdown or tolerance, so their cost depends
    # on the data
    U[0] = torch.from_numpy(M.initial_state(cfg, levels[0].grid)).to(dev)
    M.pcg64_uniform(cfg.seed, cfg.n_t, levels[0].grid.n_points, U[1:])
    eng = M._FusedCycle(levels, U, cfg.relaxation)
    eng.iteration()                     # kernel attributes set, buffers touched
    # back to the first iterate, so every phase below sees the data of the
    # solve's first V-cycle (after a converged cycle the coarse right-hand
    # sides are tiny and the corrected steps would run all K Arnoldi steps)
    U[0] = torch.from_numpy(M.initial_state(cfg, levels[0].grid)).to(dev)
    M.pcg64_uniform(cfg.seed, cfg.n_t, levels[0].grid.n_points, U[1:])
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
                          phase_bytes(levels[li], ph, li == 0)))
        walk(li + 1)
        ph = _lib.PHASE_INJ_F
        order.append((f"L{li}_{names[ph]}_{levels[li].kind}", lambda li=li, ph=ph: eng._phase(li, ph),
                      phase_bytes(levels[li], ph, li == 0)))

    walk()
    out = {}
    stream = torch.cuda.current_stream()
    for key, fn, nbytes in order:
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for _ in range(inner):
                fn()
        g.replay()
        torch.cuda.synchronize()
        ts = []
        for _ in range(reps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            g.replay()
            b.record(stream)
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b) / inner)
        ms = float(np.median(ts))
        o = out.setdefault(key, {"ms_total": 0.0, "ms_avg": ms, "bytes": nbytes, "launches": 0})
        o["ms_total"] += ms
        o["launches"] += 1
    return out, len(order) + 1   # + the norm sum


def _peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return {"hbm_gbs": float(d["hbm_gbs"]), "source": "measured (MEASURED_PEAKS.json)"}
    return {"hbm_gbs": 6650.0, "source": "fallback (B200_PROFILING.md)"}


def _ncu_fp64(dim, p):
    """FP64 instructions per node-update of the fine SL kernel (ncu-measured)."""
    path = os.path.join(ROOT, "profiles", "ncu_fp64.json")
    if not os.path.exists(path):
        return None
    with open(path) as f:
        return json.load(f).get(f"{dim}d_p{p}")


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


_ORACLE_LEVELS = {}


def _oracle_sample(name: str):
    """One V-cycle + convergence residual of the config on the host (seconds),
    plus the initial-residual time (hierarchy built once, outside the sample)."""
    import oracle as O
    kw = CONFIGS[name]
    ocfg = O.OConfig(**kw)
    if name not in _ORACLE_LEVELS:
        _ORACLE_LEVELS[name] = O.hierarchy(ocfg)
    levels = _ORACLE_LEVELS[name]
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
    t_it = time.perf_counter() - t1
    return t_r0, t_it, levels


def cpu_baseline(name: str, iters: int, samples: int = 1):
    kw = CONFIGS[name]
    n_dof = kw["n_x"] * kw["n_t"]
    best = None
    for _ in range(max(1, samples)):
        t_r0, t_it, _ = _oracle_sample(name)
        best = (t_r0, t_it) if best is None or t_it < best[1] else best
    t_r0, t_it = best
    est = t_r0 + iters * t_it
    return {"value": n_dof / est, "unit": "DOF/s", "cores": 1, "kind": "port",
            "sample": f"oracle (bit-identical numpy/C restatement of mgrit_advect): initial residual "
                      f"({t_r0:.2f}s) + one V-cycle with convergence residual ({t_it:.2f}s) of {name}, "
                      f"extrapolated x{iters} iterations; setup excluded",
            "host_cpus": os.cpu_count()}


def run_reference(args):
    rank, world, _ = _dist_env()
    if rank != 0:
        return
    kw = CONFIGS[args.config]
    gold = _golden(args.config)
    iters = gold[0]["iterations"] if gold else 19
    n_dof = kw["n_x"] * kw["n_t"]
    times = []
    for i in range(args.warmup + args.steps):
        t_r0, t_it, _ = _oracle_sample(args.config)
        if i >= args.warmup:
            times.append(t_r0 + iters * t_it)
    est = float(np.mean(times))
    value = n_dof / est
    line = {
        "impl": "reference", "metric": "MGRIT solve space-time DOF/s to 1e-10 residual", "value": value,
        "unit": "DOF/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": est * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": DESCR[args.config], "name": args.config},
        "cpu_baseline": {"value": value, "unit": "DOF/s", "cores": 1, "kind": "port",
                         "sample": f"per step: oracle initial residual + one V-cycle + residual of {args.config}, "
                                   f"extrapolated to the reference's {iters} iterations (setup excluded)",
                         "host_cpus": os.cpu_count()},
        "e2e": {"value": value, "unit": "DOF/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="cfg2", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--cpu-samples", type=int, default=1)
    ap.add_argument("--gmres-variant", default="mgs", choices=["mgs", "mgs_lowsync"],
                    help="coarse-level Arnoldi orthogonalisation (mgs = the reference's loop)")
    ap.add_argument("--launch-policy", default="auto", choices=["auto", "cta", "cluster", "auto_one"],
                    help="corrected 1D kernels: one CTA or one 8-SM cluster per row chain")
    ap.add_argument("--no-e2e", action="store_true", help="skip the host-buffer end-to-end leg")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()
