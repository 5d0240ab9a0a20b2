"""MGRIT driver and Level operator API on B200 (mirror of mgrit.py:1-390).

Same names, signatures and in-place semantics as the reference's public API
(``SolverConfig``, ``Level.step/step_batch``, ``build_hierarchy``,
``f_relax``, ``c_relax``, ``residual``, ``solve_sequential``, ``v_cycle``,
``solve``, ``sequential_reference``), but every operator application runs in
hand-written sm_100a kernels (libmgrit_b200.so) on HBM-resident state.

``solve`` uses the fused level engine (``_FusedCycle``): per level and cycle
three kernels — F+C relaxation, F-relaxation + C-point residual/restriction,
injection + post F-relaxation (+ the fine residual for the convergence test)
— captured into one CUDA graph.  The reference-structured ``v_cycle`` (one
launch per batched step, exactly mgrit.py:317-334) remains available and is
what the drop-in functions compose; both paths give identical iterates.
"""

from __future__ import annotations

import ctypes
import gc
import time
from dataclasses import dataclass, field, replace
from typing import Sequence

import numpy as np
import torch

from . import _lib
from .core import (Grid1D, Grid2D, WaveSpeed, get_wave_speed, initial_condition, pcg64_uniform,
                   require_cuda, stream_ptr, device_sum)

OPERATOR_KINDS = ("rediscretized", "corrected", "ideal", "forward_euler")
DEPARTURE_POLICIES = ("backtrack", "erk_rediscretized", "erk_substeps")
DEFAULT_CFL = 0.85
_KIND_CODE = {"fine": _lib.KIND_SL, "rediscretized": _lib.KIND_SL, "corrected": _lib.KIND_CORRECTED,
              "forward_euler": _lib.KIND_FORWARD_EULER}


GMRES_VARIANTS = ("mgs", "mgs_lowsync")
LAUNCH_POLICIES = {"auto": 0, "cta": 1, "cluster": 2, "auto_one": 3,
                   "cluster2": 4, "cluster4": 5, "cluster8": 6, "cluster16": 7}
_launch_policy = "auto"


def set_launch_policy(policy: str) -> str:
    """Kernel shape of corrected 1D phases/sweeps: "auto" (per level, the
    shape with the lowest measured cost: one CTA per row chain, two per SM
    when chains outnumber SMs, or a 2/4/8/16-CTA cluster per chain when a
    level has too few chains to fill the GPU), "auto_one" (auto without the
    two-per-SM form), "cta" (CTA kernels only), "cluster" (a cluster per
    chain whenever eligible, size by cost) or "cluster2/4/8/16" (that
    cluster size wherever eligible).  Returns the previous policy."""
    global _launch_policy
    if policy not in LAUNCH_POLICIES:
        raise ValueError(f"launch policy must be one of {sorted(LAUNCH_POLICIES)}")
    prev, _launch_policy = _launch_policy, policy
    return prev


@dataclass(frozen=True)
class GmresConfig:
    """coarse_correction.py:157-170 — tol None runs exactly max_iters iterations."""

    max_iters: int = 10
    tol: float | None = None
    # "mgs": the reference's modified Gram-Schmidt loop; "mgs_lowsync": the
    # same projection coefficients via one fused reduction per Arnoldi step
    # (Gram-corrected) on the 1D cluster kernels, where every reduction is a
    # DSMEM round trip -- equal in exact arithmetic, not bitwise
    variant: str = "mgs"

    def __post_init__(self):
        if self.max_iters < 1:
            raise ValueError("max_iters must be at least 1")
        if self.variant not in GMRES_VARIANTS:
            raise ValueError(f"gmres variant must be one of {GMRES_VARIANTS}")


@dataclass(frozen=True)
class SolverConfig:
    """mgrit.py:39-86, plus BASELINE hooks ``u0`` ("reference" | "sin4") and
    ``iterate`` ("uniform01" = reference, "pm1" = uniform [-1, 1))."""

    n_x: int
    n_t: int
    dim: int = 1
    wave_speed: str | WaveSpeed = "C1"
    p: int = 1
    r: int | None = None
    dt: float | None = None
    schedule: int | Sequence[int] = 4
    max_levels: int | None = None
    operator_kind: str = "corrected"
    departure_policy: str = "backtrack"
    gmres_mode: str | None = None
    gmres_variant: str = "mgs"
    relaxation: str = "FCF"
    seed: int = 0
    rtol: float = 1e-10
    max_iters: int = 100
    divergence_factor: float = 1e6
    u0: str = "reference"
    iterate: str = "uniform01"

    def __post_init__(self):
        if self.p % 2 == 0:
            raise ValueError("interpolation degree p must be odd")
        if self.p not in (1, 3, 5):
            raise ValueError(f"unsupported interpolation degree p={self.p}; supported: (1, 3, 5)")
        if self.operator_kind not in OPERATOR_KINDS:
            raise ValueError(f"unknown operator kind {self.operator_kind!r}")
        if self.departure_policy not in DEPARTURE_POLICIES:
            raise ValueError(f"unknown departure policy {self.departure_policy!r}")
        if self.relaxation not in ("FCF", "F"):
            raise ValueError("relaxation must be 'FCF' or 'F'")
        if self.gmres_mode not in (None, "fixed", "tolerance"):
            raise ValueError("gmres_mode must be 'fixed', 'tolerance', or None")
        if self.gmres_variant not in GMRES_VARIANTS:
            raise ValueError(f"gmres_variant must be one of {GMRES_VARIANTS}")
        if self.u0 not in ("reference", "sin4"):
            raise ValueError("u0 must be 'reference' or 'sin4'")
        if self.iterate not in ("uniform01", "pm1"):
            raise ValueError("iterate must be 'uniform01' or 'pm1'")
        speed = self.speed
        if speed.dim != self.dim:
            raise ValueError(f"wave speed {speed.name} is {speed.dim}D but config is {self.dim}D")

    @property
    def speed(self) -> WaveSpeed:
        return get_wave_speed(self.wave_speed) if isinstance(self.wave_speed, str) else self.wave_speed

    @property
    def erk_order(self) -> int:
        return self.p if self.r is None else self.r

    def schedule_factor(self, level_index: int) -> int:
        if isinstance(self.schedule, int):
            return self.schedule
        seq = list(self.schedule)
        return seq[min(level_index, len(seq) - 1)]


# ---------------------------------------------------------------------------
# device workspace shared by the operator calls


class _Workspace:
    """Per-device scratch and sticky status flag.  The status tensor of a
    device is never reallocated: captured graphs (the solve loop) keep its
    address."""

    def __init__(self):
        self.scratch: dict = {}
        self.status: dict = {}

    @staticmethod
    def _key(device) -> torch.device:
        d = torch.device(device)
        return torch.device(d.type, torch.cuda.current_device()) if d.type == "cuda" and d.index is None else d

    def get_scratch(self, nbytes: int, device) -> torch.Tensor:
        if nbytes <= 0:
            return None
        key = self._key(device)
        buf = self.scratch.get(key)
        if buf is None or buf.numel() < nbytes:
            buf = torch.empty(int(nbytes), dtype=torch.uint8, device=key)
            self.scratch[key] = buf
        return buf

    def get_status(self, device) -> torch.Tensor:
        key = self._key(device)
        st = self.status.get(key)
        if st is None:
            st = torch.zeros(1, dtype=torch.int32, device=key)
            self.status[key] = st
        return st


_WS = _Workspace()


def _ptr(t):
    return 0 if t is None else t.data_ptr()


def _check_status(device):
    st = _WS.get_status(device)
    if int(st.item()) != 0:
        st.zero_()
        raise ValueError("non-finite right-hand side in gmres_solve")


# ---------------------------------------------------------------------------
# Level


@dataclass
class Level:
    """One level of the hierarchy (mgrit.py:89-167) with device-resident records.

    ``s_x``/``s_y``: departure records [S, n_points] as the scaled periodic
    coordinate s = mod(x_dep - x_lo, L)/h (east index and eps re-derived
    exactly on every application); ``disp_x``/``disp_y``: displacements kept
    while coarser levels are built; ``sig_x``/``sig_y``: sigma fields.
    """

    index: int
    grid: Grid1D | Grid2D
    p: int
    n_steps: int
    dt: float
    kind: str
    s_x: torch.Tensor | None = None
    s_y: torch.Tensor | None = None
    disp_x: torch.Tensor | None = field(default=None, repr=False)
    disp_y: torch.Tensor | None = field(default=None, repr=False)
    sig_x: torch.Tensor | None = field(default=None, repr=False)
    sig_y: torch.Tensor | None = field(default=None, repr=False)
    gmres_cfg: GmresConfig | None = None
    cf: int | None = None
    finer: "Level | None" = None
    shared: bool = False
    stencil_numba: bool = False
    # first step whose records/sigma are stored (a time-sharded hierarchy keeps
    # only the steps its rank group works on; 0 = all steps)
    set0: int = 0
    # 2D: the records are separable (s_x independent of the mesh row, s_y of the
    # column, bitwise), so plain SL steps take the sliding-window kernel
    # (step2d.cu sl2d_sep_kernel); None = check the records on construction
    separable: bool | None = None

    def __post_init__(self):
        if self.separable is None:
            self.separable = False
            if self.grid.dim == 2 and self.s_x is not None and self.s_y is not None and self.s_x.is_cuda:
                flag = torch.zeros(1, dtype=torch.int32, device=self.s_x.device)
                rc = _lib.load().mgrit_records_separable(self.grid.n_x, self.s_x.shape[0], self.s_x.data_ptr(),
                                                         self.s_y.data_ptr(), flag.data_ptr(), stream_ptr())
                _lib.check(rc, "records_separable")
                self.separable = bool(flag.item())

    # -- read-only views of the reference's Level data (mgrit.py:89-117) -----

    @property
    def departures(self):
        """One DepartureSet view per stored record set (a single shared set for
        a constant speed), east/eps re-derived from the device records exactly
        as the kernels do; None for the ideal operator."""
        from .operators import DepartureSetView
        if self.s_x is None:
            return None
        return DepartureSetView(self)

    @property
    def sigma(self):
        """One CorrectionField (device vectors) per stored sigma set, or None."""
        from .operators import SigmaView
        return None if self.sig_x is None else SigmaView(self)

    def dep(self, n: int):
        """mgrit.py:111-112."""
        return self.departures[0 if self.shared else n]

    def sig(self, n: int):
        """mgrit.py:114-115."""
        return self.sigma[0 if self.shared else n]

    @property
    def _idx(self):
        """1D gather table (S, n_x, p+1) int32 of mgrit.py:121-126, built on demand."""
        from .operators import stencil_tables
        return stencil_tables(self)[0]

    @property
    def _w(self):
        """1D weight table (S, n_x, p+1) of mgrit.py:121-126, built on demand."""
        from .operators import stencil_tables
        return stencil_tables(self)[1]

    def desc(self, stencil_numba: bool | None = None) -> _lib.LevelDesc:
        if self.kind == "ideal":
            raise ValueError("the ideal operator is composed from the finer level")
        d = _lib.LevelDesc()
        d.dim = self.grid.dim
        d.n_x = self.grid.n_x
        d.p = self.p
        d.kind = _KIND_CODE[self.kind]
        d.shared = int(self.shared)
        d.n_steps = self.n_steps
        d.n_points = self.grid.n_points
        # kernels address step t's record at base + t * n_points: a sharded
        # level passes its base shifted by the first stored step (only the
        # stored steps are ever addressed)
        off = 0 if self.shared else self.set0 * self.grid.n_points * 8
        d.s_x = _ptr(self.s_x) - off if self.s_x is not None else 0
        d.s_y = _ptr(self.s_y) - off if self.s_y is not None else 0
        d.sig_x = _ptr(self.sig_x) - off if self.sig_x is not None else 0
        d.sig_y = _ptr(self.sig_y) - off if self.sig_y is not None else 0
        g = self.gmres_cfg or GmresConfig()
        d.gmres_max_iters = g.max_iters
        d.gmres_tol = -1.0 if g.tol is None else float(g.tol)
        d.stencil_numba = int(self.stencil_numba if stencil_numba is None else stencil_numba)
        d.gmres_lowsync = int(g.variant == "mgs_lowsync")
        d.launch_policy = LAUNCH_POLICIES[_launch_policy]
        d.sl2d_separable = int(bool(self.separable))
        return d

    @property
    def device(self):
        return self.s_x.device if self.s_x is not None else self.finer.device

    # -- operator application (mgrit.py:135-167) ----------------------------

    def _apply(self, U_in: torch.Tensor, t_first: int, t_stride: int, B: int, out: torch.Tensor,
               G: torch.Tensor | None = None, U_sub: torch.Tensor | None = None,
               t_idx: torch.Tensor | None = None, row_sumsq: torch.Tensor | None = None,
               ld_in: int | None = None, ld_out: int | None = None, ld_g: int | None = None,
               ld_sub: int | None = None, gmres_iters: torch.Tensor | None = None):
        """Thin wrapper of mgrit_apply_rows (row pointers/strides in elements)."""
        lib = _lib.load()
        n = self.grid.n_points
        d = self.desc()
        dev = U_in.device
        rows = min(B, max(1, int(lib.mgrit_resident_rows(ctypes.byref(d))) or B))
        nbytes = int(lib.mgrit_gmres_scratch_bytes(ctypes.byref(d), rows))
        scr = _WS.get_scratch(nbytes, dev)
        rc = lib.mgrit_apply_rows(
            ctypes.byref(d), B, _ptr(t_idx), t_first, t_stride,
            U_in.data_ptr(), ld_in or n, _ptr(G), ld_g or n, _ptr(U_sub), ld_sub or n,
            _ptr(out), ld_out or n, _ptr(row_sumsq), _ptr(gmres_iters), _ptr(scr),
            0 if scr is None else scr.numel(), _WS.get_status(dev).data_ptr(), stream_ptr())
        _lib.check(rc, "apply_rows")

    def step(self, n: int, u: torch.Tensor) -> torch.Tensor:
        """Advance u across step n (operator only, no forcing)."""
        u = _as_device_vec(u, self)
        if self.kind == "ideal":
            ratio = self.finer.n_steps // self.n_steps
            for k in range(ratio):
                u = self.finer.step(n * ratio + k, u)
            return u
        out = torch.empty_like(u)
        self._apply(u.reshape(1, -1), int(n), 0, 1, out.reshape(1, -1))
        if self.kind == "corrected":
            _check_status(u.device)
        return out

    def step_batch(self, t_idx, U: torch.Tensor) -> torch.Tensor:
        """Apply the steps t_idx to the matching rows of U (returns a new tensor)."""
        U = _as_device_mat(U, self)
        t = torch.as_tensor(np.asarray(t_idx, dtype=np.int64)).to(U.device)
        if self.kind == "ideal":
            ratio = self.finer.n_steps // self.n_steps
            V = U
            for k in range(ratio):
                V = self.finer.step_batch((t * ratio + k).cpu().numpy(), V)
            return V if V is not U else U.clone()
        out = torch.empty_like(U)
        if U.shape[0]:
            self._apply(U, 0, 0, U.shape[0], out, t_idx=t)
            if self.kind == "corrected":
                _check_status(U.device)
        return out


def _as_device_vec(u, lev) -> torch.Tensor:
    if isinstance(u, np.ndarray):
        u = torch.from_numpy(np.ascontiguousarray(u, dtype=np.float64)).to(lev.device)
    if u.shape[-1] != lev.grid.n_points:
        raise ValueError(f"state length {u.shape[-1]} does not match grid size {lev.grid.n_points}")
    return u.contiguous()


def _as_device_mat(U, lev) -> torch.Tensor:
    if isinstance(U, np.ndarray):
        U = torch.from_numpy(np.ascontiguousarray(U, dtype=np.float64)).to(lev.device)
    if U.shape[-1] != lev.grid.n_points:
        raise ValueError(f"state length {U.shape[-1]} does not match grid size {lev.grid.n_points}")
    return U.contiguous()


@dataclass
class ConvergenceReport:
    """mgrit.py:170-178 (+ per-phase device timings)."""

    residual_norms: np.ndarray
    iterations: int
    status: str
    final_factor: float
    wall_time: float = 0.0
    setup_time: float = 0.0
    solve_time: float = 0.0


# ---------------------------------------------------------------------------
# hierarchy construction on the device (mgrit.py:185-269, K1-K3)


def _alloc_records(S, n, dim, dev):
    s_x = torch.empty((S, n), dtype=torch.float64, device=dev)
    d_x = torch.empty_like(s_x)
    s_y = torch.empty_like(s_x) if dim == 2 else None
    d_y = torch.empty_like(s_x) if dim == 2 else None
    return s_x, s_y, d_x, d_y


def _erk(grid, speed: WaveSpeed, order, S, dt, n_sub, dt_sub, dev, set_first: int = 0):
    if speed.device is None:
        raise ValueError(f"wave speed {speed.name!r} has no device form; pass fine_coords= to build_hierarchy")
    s_x, s_y, d_x, d_y = _alloc_records(S, grid.n_points, grid.dim, dev)
    tab = _lib.erk_tableau(order)
    rc = _lib.load().mgrit_erk_departures(grid.dim, grid.n_x, _lib.SPEED_IDS[speed.device], ctypes.byref(tab),
                                          int(set_first), S, float(dt), int(n_sub), float(dt_sub), s_x.data_ptr(),
                                          _ptr(s_y), d_x.data_ptr(), _ptr(d_y), stream_ptr())
    _lib.check(rc, "erk_departures")
    return s_x, s_y, d_x, d_y


def departures_from_coords(grid, coords, dev=None):
    """Records from caller-traced departure coordinates, shape (S, n) per axis
    (DepartureSet*.from_coords, semi_lagrangian.py:175-205)."""
    dev = dev or require_cuda()
    cs = [coords] if grid.dim == 1 else list(coords)
    cs = [torch.as_tensor(np.asarray(c, dtype=np.float64)).reshape(-1, grid.n_points).to(dev) for c in cs]
    S = cs[0].shape[0]
    s_x, s_y, d_x, d_y = _alloc_records(S, grid.n_points, grid.dim, dev)
    rc = _lib.load().mgrit_departures_from_coords(grid.dim, grid.n_x, S, cs[0].data_ptr(),
                                                  _ptr(cs[1] if grid.dim == 2 else None), s_x.data_ptr(),
                                                  _ptr(s_y), d_x.data_ptr(), _ptr(d_y), stream_ptr())
    _lib.check(rc, "departures_from_coords")
    return s_x, s_y, d_x, d_y


def build_hierarchy(cfg: SolverConfig, fine_coords=None, keep_displacements: bool = False) -> list[Level]:
    """Build the level hierarchy on the device (mgrit.py:217-269).

    Fine departures come from the device ERK tracer (or ``fine_coords``,
    caller-traced departure coordinates of shape (S, n_points) per axis);
    coarse departures follow ``cfg.departure_policy``; sigma fields follow
    phi_field/sigma_accumulate.  Displacements are dropped once the next
    coarser level exists unless ``keep_displacements``.
    """
    dev = require_cuda()
    speed = cfg.speed
    if speed.dim != cfg.dim:
        raise ValueError(f"wave speed {speed.name} is {speed.dim}D but config is {cfg.dim}D")
    grid = Grid1D(cfg.n_x) if cfg.dim == 1 else Grid2D(cfg.n_x)
    dt = cfg.dt if cfg.dt is not None else DEFAULT_CFL * grid.h
    order = cfg.erk_order
    lib = _lib.load()
    shared = speed.constant
    S0 = 1 if shared else cfg.n_t
    if fine_coords is not None:
        rec = departures_from_coords(grid, fine_coords, dev)
        if rec[0].shape[0] != S0:
            raise ValueError(f"fine_coords must hold {S0} departure sets")
    else:
        rec = _erk(grid, speed, order, S0, dt, 1, dt, dev)
    fine = Level(0, grid, cfg.p, cfg.n_t, dt, "fine", rec[0], rec[1], rec[2], rec[3], shared=shared)
    levels = [fine]
    while True:
        if cfg.max_levels is not None and len(levels) >= cfg.max_levels:
            break
        prev = levels[-1]
        m = cfg.schedule_factor(len(levels) - 1)
        if prev.n_steps % m != 0 or prev.n_steps // m < 2:
            break
        n_c = prev.n_steps // m
        dt_c = prev.dt * m
        kind = cfg.operator_kind
        if kind == "ideal":
            lvl = Level(len(levels), grid, cfg.p, n_c, dt_c, "ideal", finer=prev)
        else:
            S = 1 if shared else n_c
            if cfg.departure_policy == "backtrack":
                s_x, s_y, d_x, d_y = _alloc_records(S, grid.n_points, grid.dim, dev)
                rc = lib.mgrit_backtrack(grid.dim, grid.n_x, m, S, int(prev.shared), prev.disp_x.data_ptr(),
                                         _ptr(prev.disp_y), s_x.data_ptr(), _ptr(s_y), d_x.data_ptr(),
                                         _ptr(d_y), stream_ptr())
                _lib.check(rc, "backtrack")
            elif cfg.departure_policy == "erk_rediscretized":
                s_x, s_y, d_x, d_y = _erk(grid, speed, order, S, dt_c, 1, dt_c, dev)
            else:
                n_sub = int(round(dt_c / dt))
                s_x, s_y, d_x, d_y = _erk(grid, speed, order, S, dt_c, n_sub, dt, dev)
            sig_x = sig_y = None
            if kind in ("corrected", "forward_euler"):
                sig_x = torch.empty((S, grid.n_points), dtype=torch.float64, device=dev)
                sig_y = torch.empty_like(sig_x) if grid.dim == 2 else None
                rc = lib.mgrit_phi_sigma(grid.dim, grid.n_x, cfg.p, m, S, int(prev.shared), s_x.data_ptr(),
                                         _ptr(s_y), prev.s_x.data_ptr(), _ptr(prev.s_y), _ptr(prev.sig_x),
                                         _ptr(prev.sig_y), sig_x.data_ptr(), _ptr(sig_y), stream_ptr())
                _lib.check(rc, "phi_sigma")
            lvl = Level(len(levels), grid, cfg.p, n_c, dt_c, kind, s_x, s_y, d_x, d_y, sig_x, sig_y,
                        finer=prev, shared=shared)
        prev.cf = m
        if not keep_displacements:
            prev.disp_x = prev.disp_y = None
        levels.append(lvl)
    if len(levels) < 2:
        raise ValueError("time grid does not admit any coarsening with the given schedule")
    if not keep_displacements:
        levels[-1].disp_x = levels[-1].disp_y = None
    mode = cfg.gmres_mode or ("fixed" if len(levels) == 2 else "tolerance")
    gcfg = GmresConfig(10, None if mode == "fixed" else 1e-2, cfg.gmres_variant)
    for lvl in levels[1:]:
        lvl.gmres_cfg = gcfg
    # the reference's numba sweep (mgrit.py:304-305) groups the D-stencil sum
    # differently from the numpy operator; mirror it on 1D corrected levels with >= 64 steps
    last = levels[-1]
    last.stencil_numba = (last.grid.dim == 1 and last.kind == "corrected" and last.n_steps >= 64)
    return levels


# ---------------------------------------------------------------------------
# relaxation, residual, cycling — reference-structured (mgrit.py:276-334)


def _rows(U: torch.Tensor, start: int, step: int, count: int):
    return U[start: start + step * (count - 1) + 1: step] if count > 0 else U[start:start]


def f_relax(level: Level, U, G, m: int | None = None) -> None:
    """mgrit.py:276-283 (in place; one batched launch per F-point offset)."""
    U, G, wb = _io(level, U, G)
    m = level.cf if m is None else m
    N = level.n_steps
    n_starts = (N + m - 1) // m
    for k in range(1, m):
        B = n_starts
        if (n_starts - 1) * m + k > N:
            raise IndexError(f"f_relax: step index {(n_starts - 1) * m + k} out of bounds for {N} steps")
        _step_rows_strided(level, U, G, k - 1, m, B)
    wb()


def c_relax(level: Level, U, G, m: int | None = None) -> None:
    """mgrit.py:286-290."""
    U, G, wb = _io(level, U, G)
    m = level.cf if m is None else m
    B = level.n_steps // m
    _step_rows_strided(level, U, G, m - 1, m, B)
    wb()


def _step_rows_strided(level, U, G, first, stride, B):
    """U[first + b*stride + 1] = Phi U[first + b*stride] + G[...] for b < B."""
    if B <= 0:
        return
    n = level.grid.n_points
    if level.kind == "ideal":
        t = np.arange(B) * stride + first
        V = level.step_batch(t, U[first: first + stride * (B - 1) + 1: stride])
        U[first + 1: first + 1 + stride * (B - 1) + 1: stride] = V + G[first + 1: first + 1 + stride * (B - 1) + 1: stride]
        return
    level._apply(U[first:], first, stride, B, U[first + 1:], G=G[first + 1:], ld_in=stride * n,
                 ld_out=stride * n, ld_g=stride * n)
    if level.kind == "corrected":
        _check_status(U.device)


def residual(level: Level, U, G):
    """r_n = g_n + Phi u_{n-1} - u_n, r_0 = 0 (mgrit.py:293-299); new tensor."""
    host = isinstance(U, np.ndarray)
    U, G, _ = _io(level, U, G)
    R = torch.empty_like(U)
    R[0] = 0.0
    N = level.n_steps
    if level.kind == "ideal":
        R[1:] = (G[1:] + level.step_batch(np.arange(N), U[:-1])) - U[1:]
    else:
        level._apply(U, 0, 1, N, R[1:], G=G[1:], U_sub=U[1:])
        if level.kind == "corrected":
            _check_status(U.device)
    return R.cpu().numpy() if host else R


def solve_sequential(level: Level, U, G) -> None:
    """Exact sequential solve of a level (mgrit.py:302-314; numba sweep grouping
    for 1D corrected levels with >= 64 steps)."""
    U, G, wb = _io(level, U, G)
    if level.kind == "ideal":
        for n in range(1, level.n_steps + 1):
            U[n] = level.step(n - 1, U[n - 1]) + G[n]
        wb()
        return
    _sweep(level, U, G, zero_init=False)
    wb()


def _sweep(level: Level, U: torch.Tensor, G: torch.Tensor | None, zero_init: bool, numba=None):
    lib = _lib.load()
    numba = (level.grid.dim == 1 and level.kind == "corrected" and level.n_steps >= 64) if numba is None else numba
    d = level.desc(stencil_numba=numba)
    nbytes = int(lib.mgrit_gmres_scratch_bytes(ctypes.byref(d), 1))
    scr = _WS.get_scratch(nbytes, U.device)
    n = level.grid.n_points
    rc = lib.mgrit_sequential_sweep(ctypes.byref(d), U.data_ptr(), n, _ptr(G), n, int(zero_init), 0, _ptr(scr),
                                    0 if scr is None else scr.numel(), _WS.get_status(U.device).data_ptr(),
                                    stream_ptr())
    _lib.check(rc, "sequential_sweep")


def _io(level, U, G):
    """Accept numpy (copied to the device and written back) or device tensors."""
    if isinstance(U, np.ndarray):
        dev = level.device
        Ud = torch.from_numpy(np.ascontiguousarray(U)).to(dev)
        Gd = torch.from_numpy(np.ascontiguousarray(G)).to(dev)

        def wb():
            U[...] = Ud.cpu().numpy()
        return Ud, Gd, wb
    if not U.is_contiguous() or (G is not None and not G.is_contiguous()):
        raise ValueError("U and G must be contiguous (n_rows, n_points) float64 tensors")
    return U, G, (lambda: None)


def v_cycle(levels: list[Level], li: int, U, G, relaxation: str = "FCF") -> None:
    """One recursive V-cycle (mgrit.py:317-334), reference-structured."""
    U, G, wb = _io(levels[li], U, G)
    lev = levels[li]
    if li == len(levels) - 1:
        solve_sequential(lev, U, G)
        wb()
        return
    m = lev.cf
    f_relax(lev, U, G)
    if relaxation == "FCF":
        c_relax(lev, U, G)
        f_relax(lev, U, G)
    R = residual(lev, U, G)
    Gc = R[::m].contiguous()
    Uc = torch.zeros((lev.n_steps // m + 1, lev.grid.n_points), dtype=torch.float64, device=U.device)
    v_cycle(levels, li + 1, Uc, Gc, relaxation)
    U[::m] += Uc
    f_relax(lev, U, G)
    wb()


# ---------------------------------------------------------------------------
# fused engine


class _FusedCycle:
    """Device buffers + launch sequence of one V-cycle using the fused phase
    kernels (1D, non-ideal levels)."""

    def __init__(self, levels: list[Level], U: torch.Tensor, relaxation: str):
        self.levels = levels
        self.relaxation = relaxation
        self.dev = U.device
        n = levels[0].grid.n_points
        L = len(levels)
        self.U = [U] + [torch.zeros((lv.n_steps + 1, n), dtype=torch.float64, device=self.dev) for lv in levels[1:]]
        self.G = [None] + [torch.zeros((lv.n_steps + 1, n), dtype=torch.float64, device=self.dev) for lv in levels[1:]]
        self.C = [torch.zeros((lv.n_steps // lv.cf + 1, n), dtype=torch.float64, device=self.dev)
                  for lv in levels[:-1]]
        self.partial = torch.zeros(levels[0].n_steps // levels[0].cf, dtype=torch.float64, device=self.dev)
        self.sumsq = torch.zeros(1, dtype=torch.float64, device=self.dev)
        self.status = _WS.get_status(self.dev)
        lib = _lib.load()
        self.descs = [lv.desc() for lv in levels[:-1]]
        self.desc_last = levels[-1].desc(stencil_numba=levels[-1].stencil_numba)
        need = 0
        for lv, d in zip(levels[:-1], self.descs):
            rows = min(lv.n_steps // lv.cf, max(1, int(lib.mgrit_resident_rows(ctypes.byref(d)))))
            need = max(need, int(lib.mgrit_gmres_scratch_bytes(ctypes.byref(d), rows)))
        need = max(need, int(lib.mgrit_gmres_scratch_bytes(ctypes.byref(self.desc_last), 1)))
        self.scratch = torch.empty(max(need, 8), dtype=torch.uint8, device=self.dev)
        self._args = {}
        for li in range(L - 1):
            for ph in (_lib.PHASE_FC, _lib.PHASE_F_RES, _lib.PHASE_FONLY_RES, _lib.PHASE_INJ_F):
                self._args[(li, ph)] = self._make_args(li, ph)
        # The reference's V-cycle ends with an F-relaxation of the fine level
        # (mgrit.py:334) and the next one starts with the same F-relaxation
        # (mgrit.py:325) of unchanged C-points: identical rows.  The fine FC
        # phase therefore runs only its C-step; prologue() establishes the
        # invariant before the first V-cycle.  2D: the phase launch skips its
        # batched F-steps (mgrit_phase_args::f_relaxed).  1D: the C-step is one
        # batched row launch (U[(c+1)m - 1] -> Cbuf[c + 1] for every interval)
        # instead of the fused phase kernel, which would walk the interval again.
        self.skip_f = relaxation == "FCF" and L > 1 and levels[0].kind != "ideal"
        if self.skip_f:
            self._fc_full = self._make_args(0, _lib.PHASE_FC)
            self._args[(0, _lib.PHASE_FC)].f_relaxed = 1

    def _make_args(self, li, phase):
        lv = self.levels[li]
        n = lv.grid.n_points
        a = _lib.PhaseArgs()
        a.phase = phase
        a.m = lv.cf
        a.c_begin = 0
        a.c_count = lv.n_steps // lv.cf
        a.n_intervals = lv.n_steps // lv.cf
        a.U = self.U[li].data_ptr(); a.ldu = n; a.u_row0 = 0
        a.G = _ptr(self.G[li]); a.ldg = n; a.g_row0 = 0
        a.Cbuf = self.C[li].data_ptr()
        a.Uc = self.U[li + 1].data_ptr()
        a.Gc = self.G[li + 1].data_ptr() if phase in (_lib.PHASE_F_RES, _lib.PHASE_FONLY_RES) else 0
        a.c_row0 = 0
        a.partial = self.partial.data_ptr() if (li == 0 and phase == _lib.PHASE_INJ_F) else 0
        a.partial0 = 0
        a.zero_init = int(li > 0)
        return a

    def _phase(self, li, phase):
        lib = _lib.load()
        if li == 0 and phase == _lib.PHASE_FC and self.skip_f and self.levels[0].grid.dim == 1:
            lv = self.levels[0]
            n, m = lv.grid.n_points, lv.cf
            U = self.U[0]
            lv._apply(U[m - 1:], m - 1, m, lv.n_steps // m, self.C[0][1:], ld_in=m * n, ld_out=n)
            return
        rc = lib.mgrit_level_phase(ctypes.byref(self.descs[li]), ctypes.byref(self._args[(li, phase)]),
                                   self.scratch.data_ptr(), self.scratch.numel(), self.status.data_ptr(),
                                   stream_ptr())
        _lib.check(rc, "level_phase")

    def prologue(self):
        """F-relax the fine level once before the first V-cycle (see skip_f)."""
        if self.skip_f:
            lib = _lib.load()
            rc = lib.mgrit_level_phase(ctypes.byref(self.descs[0]), ctypes.byref(self._fc_full),
                                       self.scratch.data_ptr(), self.scratch.numel(), self.status.data_ptr(),
                                       stream_ptr())
            _lib.check(rc, "level_phase")

    def cycle(self, li: int = 0):
        if li == len(self.levels) - 1:
            lib = _lib.load()
            n = self.levels[li].grid.n_points
            rc = lib.mgrit_sequential_sweep(ctypes.byref(self.desc_last), self.U[li].data_ptr(), n,
                                            self.G[li].data_ptr(), n, 1, 0, self.scratch.data_ptr(),
                                            self.scratch.numel(), self.status.data_ptr(), stream_ptr())
            _lib.check(rc, "sequential_sweep")
            return
        if self.relaxation == "FCF":
            self._phase(li, _lib.PHASE_FC)
            self._phase(li, _lib.PHASE_F_RES)
        else:
            self._phase(li, _lib.PHASE_FONLY_RES)
        self.cycle(li + 1)
        self._phase(li, _lib.PHASE_INJ_F)

    def iteration(self):
        """One V-cycle + fine residual norm^2 into self.sumsq (device)."""
        self.cycle(0)
        _lib.check(_lib.load().mgrit_sum(self.partial.data_ptr(), self.partial.numel(), self.sumsq.data_ptr(),
                                         stream_ptr()), "sum")


def _fused_ok(levels):
    return all(lv.kind != "ideal" for lv in levels)


def initial_state(cfg: SolverConfig, grid) -> np.ndarray:
    return initial_condition(grid, cfg.u0)


def solve(cfg: SolverConfig, levels: list[Level] | None = None, *, initial_iterate=None,
          output: str = "numpy", out=None, use_graph: bool = True, engine: str = "auto"):
    """Run MGRIT (mgrit.py:337-378) on the device.

    ``initial_iterate``: optional host array (n_t, n_points) uploaded as U[1:];
    by default U[1:] is numpy's ``default_rng(seed).random`` stream generated
    bit-identically on the device (``iterate="pm1"`` maps it to [-1, 1)).
    ``output``: "numpy" (reference behaviour, host copy of U) or "device".
    ``out``: optional preallocated host buffer (numpy array or pinned torch
    CPU tensor) of shape (n_t + 1, n_points) receiving U; returned as numpy.
    ``engine``: "fused" (default when supported), "reference" (the
    reference-structured v_cycle built from batched launches).
    """
    t_begin = time.perf_counter()
    dev = require_cuda()
    if levels is None:
        levels = build_hierarchy(cfg)
    torch.cuda.synchronize()
    t_setup = time.perf_counter() - t_begin
    t_solve0 = time.perf_counter()
    fine = levels[0]
    grid = fine.grid
    n = grid.n_points
    use_fused = (engine == "fused") or (engine == "auto" and _fused_ok(levels))
    if use_fused and not _fused_ok(levels):
        raise ValueError("fused engine needs a hierarchy without ideal levels")
    sess = _session(levels, cfg, dev) if use_fused else None
    U = sess.U if sess is not None else torch.empty((cfg.n_t + 1, n), dtype=torch.float64, device=dev)
    U[0] = _initial_row(cfg, fine, dev)
    if initial_iterate is not None:
        src = torch.as_tensor(initial_iterate)
        U[1:].copy_(src.reshape(cfg.n_t, n), non_blocking=True)
    else:
        pcg64_uniform(cfg.seed, cfg.n_t, n, U[1:], pm1=(cfg.iterate == "pm1"))
    status = _WS.get_status(dev)
    status.zero_()

    # initial residual r0 (all rows: the random iterate has F-point residuals);
    # only the per-row sums of squares are produced (no residual array)
    row_ss = sess.row_ss if sess is not None else torch.empty(cfg.n_t, dtype=torch.float64, device=dev)
    fine._apply(U, 0, 1, cfg.n_t, None, U_sub=U[1:], row_sumsq=row_ss)
    r0_ss = device_sum(row_ss)
    state = "max_iters"
    G0 = torch.zeros_like(U) if not use_fused else None

    if use_fused and cfg.max_iters >= 1:
        sess.engine.prologue()
    if use_fused and use_graph and cfg.max_iters >= 1:
        # device-resident loop: one graph launch, one host sync per solve
        loop = _solve_loop(sess, cfg, status)
        lib = _lib.load()
        _lib.check(lib.mgrit_loop_init(r0_ss.data_ptr(), loop.hist.data_ptr(), loop.ctrl.data_ptr(),
                                       loop.par.data_ptr(), float(cfg.rtol), float(cfg.divergence_factor),
                                       int(cfg.max_iters), stream_ptr()), "loop_init")
        _lib.check(lib.mgrit_loop_launch(loop.handle, stream_ptr()), "loop_launch")
        ctrl = loop.ctrl.cpu()
        k = int(ctrl[0])
        state = _lib.LOOP_STATES[int(ctrl[1])]
        history = loop.hist[:k + 1].cpu().tolist()
    elif use_fused:
        history = [float(torch.sqrt(r0_ss).item())]
        r0 = history[0]
        eng = sess.engine
        for it in range(cfg.max_iters):
            eng.iteration()
            ss = float(eng.sumsq.item())
            bad = int(status.item())
            if bad:
                history.append(float("nan"))
                state = "diverged"
                break
            r = float(np.sqrt(ss))
            history.append(r)
            if not np.isfinite(r) or r >= cfg.divergence_factor * r0:
                state = "diverged"
                break
            if r <= cfg.rtol * r0:
                state = "converged"
                break
    else:
        history = [float(torch.sqrt(r0_ss).item())]
        r0 = history[0]
        for _ in range(cfg.max_iters):
            try:
                v_cycle(levels, 0, U, G0, cfg.relaxation)
                Rf = residual(fine, U, G0)
                r = float(torch.sqrt(device_sum(torch.square(Rf).reshape(-1))).item())
            except (ValueError, FloatingPointError):
                history.append(float("nan"))
                state = "diverged"
                break
            history.append(r)
            if not np.isfinite(r) or r >= cfg.divergence_factor * r0:
                state = "diverged"
                break
            if r <= cfg.rtol * r0:
                state = "converged"
                break
    if out is not None:
        dst = torch.from_numpy(out) if isinstance(out, np.ndarray) else out
        dst.copy_(U)
        result = dst.numpy()
    elif output == "numpy":
        result = U.cpu().numpy()
    else:
        result = U.clone() if sess is not None else U
    torch.cuda.synchronize()
    t_end = time.perf_counter()
    hist = np.array(history)
    factor = float(hist[-1] / hist[-2]) if len(hist) > 1 else float("nan")
    rep = ConvergenceReport(hist, len(hist) - 1, state, factor, t_end - t_begin, t_setup, t_end - t_solve0)
    return rep, result


@dataclass
class _Session:
    """Per-hierarchy solve workspace: the state buffer, the fused engine and
    its captured solve loop survive across solve() calls on the same levels."""

    U: torch.Tensor
    row_ss: torch.Tensor
    engine: "_FusedCycle"
    loop: "_Loop | None" = None


# Loops whose owner was garbage-collected.  They are destroyed only at a safe
# point (_flush_loops, outside any stream capture): the cyclic GC can run a
# finaliser while another loop is being captured, and destroying a graph
# during a capture invalidates that capture.
_DEAD_LOOPS: list = []


def _flush_loops():
    while _DEAD_LOOPS:
        _lib.load().mgrit_loop_destroy(_DEAD_LOOPS.pop())


class _Loop:
    """The captured device-resident convergence loop (loop.cu): a CUDA graph
    whose WHILE node runs one V-cycle + the stop test per pass."""

    def __init__(self, handle, hist, ctrl, par):
        self.handle, self.hist, self.ctrl, self.par = handle, hist, ctrl, par

    def __del__(self):
        if self.handle:
            _DEAD_LOOPS.append(self.handle)
            self.handle = None


def _solve_loop(sess: _Session, cfg: SolverConfig, status: torch.Tensor) -> _Loop:
    """Capture (once per session, again only if max_iters outgrows the
    history buffer) the V-cycle + stop test into the body of a WHILE node."""
    if sess.loop is not None and sess.loop.hist.numel() > cfg.max_iters:
        return sess.loop
    sess.loop = None
    _flush_loops()
    lib = _lib.load()
    dev = sess.U.device
    eng = sess.engine
    hist = torch.zeros(max(cfg.max_iters, 100) + 1, dtype=torch.float64, device=dev)
    ctrl = torch.zeros(4, dtype=torch.int32, device=dev)
    par = torch.zeros(2, dtype=torch.float64, device=dev)
    cur = torch.cuda.current_stream()
    side = torch.cuda.Stream(device=dev)   # the legacy default stream cannot be captured
    side.wait_stream(cur)
    h = ctypes.c_void_p()
    gc_was_enabled = gc.isenabled()
    gc.disable()   # no finalisers (CUDA frees) on this thread while capturing
    try:
        with torch.cuda.stream(side):
            sp = stream_ptr()
            _lib.check(lib.mgrit_loop_begin(sp, ctypes.byref(h)), "loop_begin")
            try:
                eng.iteration()
                _lib.check(lib.mgrit_loop_check(h, eng.sumsq.data_ptr(), status.data_ptr(), hist.data_ptr(),
                                                ctrl.data_ptr(), par.data_ptr(), sp), "loop_check")
                _lib.check(lib.mgrit_loop_end(h, sp), "loop_end")
            except Exception:
                lib.mgrit_loop_destroy(h)
                raise
    finally:
        if gc_was_enabled:
            gc.enable()
    cur.wait_stream(side)
    sess.loop = _Loop(h, hist, ctrl, par)
    sess.loop.body_kernels = int(lib.mgrit_loop_body_kernels(h))
    return sess.loop


def _initial_row(cfg: SolverConfig, fine: "Level", dev) -> torch.Tensor:
    """U[0] = u0 on the grid (mgrit.py:352), computed on the host with numpy
    (the reference's values, bit for bit) once per hierarchy and kept in HBM."""
    cache = fine.__dict__.setdefault("_u0_rows", {})
    row = cache.get(cfg.u0)
    if row is None or row.device != dev:
        row = torch.from_numpy(initial_state(cfg, fine.grid)).to(dev)
        cache[cfg.u0] = row
    return row


def _session(levels, cfg, dev) -> _Session:
    key = (cfg.n_t, cfg.relaxation, _launch_policy,
           tuple((lv.kind, lv.gmres_cfg, lv.stencil_numba) for lv in levels))
    cache = levels[0].__dict__.setdefault("_sessions", {})
    sess = cache.get(key)
    if sess is None:
        n = levels[0].grid.n_points
        U = torch.empty((cfg.n_t + 1, n), dtype=torch.float64, device=dev)
        sess = _Session(U, torch.empty(cfg.n_t, dtype=torch.float64, device=dev),
                        _FusedCycle(levels, U, cfg.relaxation))
        cache[key] = sess
    return sess


def _capture(fn):
    """Capture ``fn``'s launches (all on the current stream) in a CUDA graph."""
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    return g


def sequential_reference(cfg: SolverConfig, levels: list[Level] | None = None, output: str = "numpy"):
    """Plain sequential time stepping of the fine level (mgrit.py:381-390) —
    also the sequential GPU time-stepping baseline (one CTA walks all steps)."""
    dev = require_cuda()
    if levels is None:
        levels = build_hierarchy(replace(cfg, max_levels=2))
    fine = levels[0]
    U = torch.empty((cfg.n_t + 1, fine.grid.n_points), dtype=torch.float64, device=dev)
    U[0] = torch.from_numpy(initial_state(cfg, fine.grid)).to(dev)
    _sweep(fine, U, None, zero_init=False)
    return U.cpu().numpy() if output == "numpy" else U
