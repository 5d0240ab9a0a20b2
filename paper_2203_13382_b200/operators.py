"""Operator-level API of the reference below ``Level`` (mgrit_advect/__init__.py:
8-16): the semi-Lagrangian step, the truncation-error-corrected and
forward-Euler coarse steps, ``apply_ImSD``, ``gmres_solve``, ``decompose``,
``interp_weights`` and the ``DepartureSet`` / ``CorrectionField`` records, with
the reference's signatures, argument meaning and errors, backed by the
sm_100a kernels of libmgrit_b200.so.

Inputs may be numpy arrays (the reference's types; results come back as
numpy) or CUDA tensors (results stay on the device).  A reference
``DepartureSet1D/2D`` (or one of ours) is accepted as is: its ``east``/``eps``
(2D: ``east_x``/``eps``, ``east_y``/``nu``) become device records through
``mgrit_records_from_east_eps``, which reproduces those exact (east, eps) on
every application.

``gmres_solve`` runs on the device for the coarse-correction operator
(``ImSD(field, stencil, grid)``, or the reference's own
``lambda v: apply_ImSD(field, stencil, v, grid)`` rewritten as that object);
an arbitrary Python callable has no device form and is rejected (no CPU
fallback on the product path).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .core import Grid1D, Grid2D, require_cuda, stream_ptr
from .mgrit import GmresConfig, Level, _WS, _check_status

SUPPORTED_DEGREES = (1, 3, 5)


def _check_degree(p: int) -> None:
    if p not in SUPPORTED_DEGREES:
        raise ValueError(f"unsupported interpolation degree p={p}; supported: {SUPPORTED_DEGREES}")


def stencil_extents(p: int) -> tuple[int, int]:
    """semi_lagrangian.py:26-29."""
    _check_degree(p)
    return (p + 1) // 2, (p - 1) // 2


@dataclass(frozen=True)
class ErkScheme:
    """semi_lagrangian.py:32-43."""

    order: int
    a: np.ndarray
    b: np.ndarray
    c: np.ndarray

    @property
    def n_stages(self) -> int:
        return len(self.b)


def erk_scheme(order: int) -> ErkScheme:
    """The tracing tableaux (semi_lagrangian.py:46-72), same constants as the
    device tracer uses."""
    t = _lib.erk_tableau(order)
    s = t.n_stages
    a = np.array(t.a[:]).reshape(6, 6)[:s, :s].copy()
    return ErkScheme(order, a, np.array(t.b[:s]), np.array(t.c[:s]))


def derivative_stencil(p: int) -> np.ndarray:
    """coarse_correction.py:35-47."""
    _check_degree(p)
    return {1: np.array([1.0, -2.0, 1.0]), 3: np.array([1.0, -4.0, 6.0, -4.0, 1.0]),
            5: np.array([1.0, -6.0, 15.0, -20.0, 15.0, -6.0, 1.0])}[p]


def _degree_of_stencil(stencil) -> int:
    st = np.asarray(stencil, dtype=float)
    for p in SUPPORTED_DEGREES:
        if st.shape == (p + 2,) and np.array_equal(st, derivative_stencil(p)):
            return p
    raise ValueError("the device correction operator supports derivative_stencil(p), p in (1, 3, 5)")


# ---------------------------------------------------------------------------
# host/device plumbing


def _dev(x, dtype=torch.float64) -> torch.Tensor:
    if isinstance(x, torch.Tensor):
        return x.to(device=require_cuda() if not x.is_cuda else x.device, dtype=dtype).contiguous()
    return torch.from_numpy(np.ascontiguousarray(np.asarray(x), dtype=np.float64 if dtype == torch.float64
                                                 else np.int64)).to(require_cuda())


def _out(t: torch.Tensor, like):
    return t if isinstance(like, torch.Tensor) else t.cpu().numpy()


# ---------------------------------------------------------------------------
# records


@dataclass
class DepartureSet1D:
    """semi_lagrangian.py:164-183: east index, offset eps in [0, 1) and the
    unwrapped displacement arrival - departure of every node."""

    t_start: float
    dt: float
    east: np.ndarray
    eps: np.ndarray
    displacement: np.ndarray | None

    @classmethod
    def from_coords(cls, grid: Grid1D, arrival, coords, t_start: float, dt: float) -> "DepartureSet1D":
        east, eps = decompose(grid, coords)
        return cls(t_start, dt, east, eps, arrival - coords)


@dataclass
class DepartureSet2D:
    """semi_lagrangian.py:186-205 (flat, x fastest)."""

    t_start: float
    dt: float
    east_x: np.ndarray
    east_y: np.ndarray
    eps: np.ndarray
    nu: np.ndarray
    displacement_x: np.ndarray | None
    displacement_y: np.ndarray | None

    @classmethod
    def from_coords(cls, grid: Grid2D, arrival_x, arrival_y, coords_x, coords_y, t_start: float,
                    dt: float) -> "DepartureSet2D":
        ax = grid.axis
        east_x, eps = decompose(ax, coords_x)
        east_y, nu = decompose(ax, coords_y)
        return cls(t_start, dt, east_x, east_y, eps, nu, arrival_x - coords_x, arrival_y - coords_y)


@dataclass
class CorrectionField:
    """coarse_correction.py:69-89."""

    x: np.ndarray
    y: np.ndarray | None = None

    @property
    def dim(self) -> int:
        return 1 if self.y is None else 2

    def __add__(self, other: "CorrectionField") -> "CorrectionField":
        if self.dim != other.dim:
            raise ValueError("cannot add correction fields of different dimensions")
        if self.y is None:
            return CorrectionField(self.x + other.x)
        return CorrectionField(self.x + other.x, self.y + other.y)


def _axis_n(grid) -> int:
    return grid.n_x


def records_from_departures(grid, departures) -> tuple[torch.Tensor, torch.Tensor | None]:
    """Device records s (1, n_points) per axis from a DepartureSet's (east, eps)."""
    lib = _lib.load()
    n_x = _axis_n(grid)
    if hasattr(departures, "nu"):
        pairs = [(departures.east_x, departures.eps), (departures.east_y, departures.nu)]
    else:
        pairs = [(departures.east, departures.eps)]
    out = []
    for east, eps in pairs:
        e = _dev(east, torch.int64)
        x = _dev(eps)
        if e.numel() != grid.n_points or x.numel() != grid.n_points:
            raise ValueError(f"departure set size does not match grid size {grid.n_points}")
        s = torch.empty((1, grid.n_points), dtype=torch.float64, device=x.device)
        _lib.check(lib.mgrit_records_from_east_eps(n_x, e.numel(), e.data_ptr(), x.data_ptr(), s.data_ptr(),
                                                   stream_ptr()), "records_from_east_eps")
        out.append(s)
    return out[0], (out[1] if len(out) == 2 else None)


def decompose(grid, coords):
    """(east neighbour index mod n_x, eps in [0, 1)) of coordinates on a
    periodic axis (semi_lagrangian.py:118-137), on the device."""
    c = _dev(coords)
    east = torch.empty(c.shape, dtype=torch.int64, device=c.device)
    eps = torch.empty_like(c)
    _lib.check(_lib.load().mgrit_decompose(grid.n_x, c.numel(), c.data_ptr(), east.data_ptr(), eps.data_ptr(),
                                           stream_ptr()), "decompose")
    return _out(east, coords), _out(eps, coords)


def interp_weights(p: int, eps):
    """Lagrange weights over offsets -l..r at -eps, shape (len(eps), p+1)
    (semi_lagrangian.py:140-161), on the device."""
    _check_degree(p)
    e = _dev(eps).reshape(-1)
    w = torch.empty((e.numel(), p + 1), dtype=torch.float64, device=e.device)
    _lib.check(_lib.load().mgrit_interp_weights(p, e.numel(), e.data_ptr(), w.data_ptr(), stream_ptr()),
               "interp_weights")
    return _out(w, eps)


# ---------------------------------------------------------------------------
# operators


def _one_step_level(grid, departures, p, kind, field=None, cfg: GmresConfig | None = None) -> Level:
    _check_degree(p)
    s_x, s_y = records_from_departures(grid, departures)
    sig_x = sig_y = None
    if field is not None:
        sig_x = _dev(field.x).reshape(1, -1)
        if grid.dim == 2:
            if field.y is None:
                raise ValueError("2D correction needs the y coefficient vector")
            sig_y = _dev(field.y).reshape(1, -1)
        if sig_x.shape[1] != grid.n_points:
            raise ValueError("correction field and state shapes differ")
    dt = float(getattr(departures, "dt", 0.0))
    return Level(0, grid, p, 1, dt, kind, s_x, s_y, sig_x=sig_x, sig_y=sig_y, gmres_cfg=cfg)


def _state(u, grid):
    if u.shape[-1] != grid.n_points:
        raise ValueError(f"state length {u.shape[-1]} does not match grid size {grid.n_points}")
    return _dev(u)


def sl_step(grid, departures, p: int, u):
    """One semi-Lagrangian step: interpolate u at the departure points
    (semi_lagrangian.py:220-227, 238-253); bit-identical to the reference."""
    v = _state(u, grid)
    lv = _one_step_level(grid, departures, p, "fine")
    return _out(lv.step(0, v), u)


def corrected_coarse_step(grid, departures, p: int, field: CorrectionField, cfg: GmresConfig, u):
    """SL step followed by GMRES on (I - diag(field) D) x = S u
    (coarse_correction.py:231-240)."""
    v = _state(u, grid)
    lv = _one_step_level(grid, departures, p, "corrected", field, _gmres_cfg(cfg))
    return _out(lv.step(0, v), u)


def forward_euler_coarse_step(grid, departures, p: int, field: CorrectionField, u):
    """SL step followed by I + diag(field) D (coarse_correction.py:243-254)."""
    v = _state(u, grid)
    lv = _one_step_level(grid, departures, p, "forward_euler", field)
    return _out(lv.step(0, v), u)


def _gmres_cfg(cfg) -> GmresConfig:
    if isinstance(cfg, GmresConfig):
        return cfg
    return GmresConfig(int(cfg.max_iters), None if cfg.tol is None else float(cfg.tol))


def _grid_for(v, grid, dim):
    if grid is not None:
        return grid
    if dim == 2:
        raise ValueError("apply_ImSD needs the grid in 2D")
    return Grid1D(int(v.shape[-1]))


def apply_ImSD(field: CorrectionField, stencil, v, grid=None):
    """(I - diag(field) D) v (coarse_correction.py:130-149), bit-identical."""
    vx = _dev(v)
    sx = _dev(field.x)
    if sx.shape != vx.shape:
        raise ValueError("correction field and state shapes differ")
    p = _degree_of_stencil(stencil)
    g = _grid_for(vx, grid, field.dim)
    sy = _dev(field.y) if field.dim == 2 else None
    out = torch.empty_like(vx)
    _lib.check(_lib.load().mgrit_apply_imsd(field.dim, g.n_x, p, 1, sx.data_ptr(), 0 if sy is None else sy.data_ptr(),
                                            vx.data_ptr(), vx.numel(), out.data_ptr(), out.numel(), stream_ptr()),
               "apply_imsd")
    return _out(out, v)


def apply_IpSD(field: CorrectionField, stencil, v, grid=None):
    """2 v - (I - diag(field) D) v (coarse_correction.py:152-154)."""
    vx = _dev(v)
    return _out(2.0 * vx - _dev(apply_ImSD(field, stencil, vx, grid)), v)


@dataclass(frozen=True)
class ImSD:
    """The coarse-correction operator v -> (I - diag(field) D) v as an object
    gmres_solve can run on the device (the reference passes the equivalent
    lambda, coarse_correction.py:237)."""

    field: CorrectionField
    stencil: np.ndarray
    grid: Grid1D | Grid2D | None = None

    def __call__(self, v):
        return apply_ImSD(self.field, self.stencil, v, self.grid)


def _identity_records(grid) -> tuple[torch.Tensor, torch.Tensor | None]:
    """s = node index on every axis: east = i, eps = 0, so the SL gather is
    exactly the identity (weights 1 and +-0) and a corrected step reduces to
    the GMRES solve of its right-hand side."""
    dev = require_cuda()
    n = grid.n_x
    ix = torch.arange(n, dtype=torch.float64, device=dev)
    if grid.dim == 1:
        return ix.reshape(1, -1), None
    return ix.repeat(n).reshape(1, -1), ix.repeat_interleave(n).reshape(1, -1)


def gmres_solve(apply_op, rhs, cfg):
    """Non-restarted MGS-GMRES with zero initial guess for the correction
    operator (coarse_correction.py:173-228); returns (x, residual-norm
    history).  Raises ValueError on a non-finite right-hand side."""
    if not isinstance(apply_op, ImSD):
        raise TypeError("device gmres_solve runs the coarse-correction operator: pass "
                        "ImSD(field, stencil, grid) (no host fallback for arbitrary callables)")
    r = _dev(rhs)
    gc = _gmres_cfg(cfg)
    grid = _grid_for(r, apply_op.grid, apply_op.field.dim)
    p = _degree_of_stencil(apply_op.stencil)
    s_x, s_y = _identity_records(grid)
    sig_x = _dev(apply_op.field.x).reshape(1, -1)
    sig_y = _dev(apply_op.field.y).reshape(1, -1) if apply_op.field.dim == 2 else None
    lv = Level(0, grid, p, 1, 0.0, "corrected", s_x, s_y, sig_x=sig_x, sig_y=sig_y, gmres_cfg=gc)
    lib = _lib.load()
    d = lv.desc()
    x = torch.empty((1, grid.n_points), dtype=torch.float64, device=r.device)
    iters = torch.zeros(1, dtype=torch.int32, device=r.device)
    hist = torch.zeros((1, gc.max_iters + 1), dtype=torch.float64, device=r.device)
    nbytes = int(lib.mgrit_gmres_scratch_bytes(ctypes.byref(d), 1))
    scr = _WS.get_scratch(nbytes, r.device)
    _lib.check(lib.mgrit_apply_rows_hist(ctypes.byref(d), 1, None, 0, 0, r.data_ptr(), grid.n_points, x.data_ptr(),
                                         grid.n_points, iters.data_ptr(), hist.data_ptr(),
                                         0 if scr is None else scr.data_ptr(), 0 if scr is None else scr.numel(),
                                         _WS.get_status(r.device).data_ptr(), stream_ptr()), "gmres_solve")
    _check_status(r.device)
    k = int(iters.item())
    h = hist[0, :k + 1] if k > 0 else hist[0, :1]
    return _out(x.reshape(r.shape), rhs), _out(h, rhs)


# ---------------------------------------------------------------------------
# Level data views (mgrit.py:89-126)


class DepartureSetView:
    """Read-only sequence of a level's departure sets as DepartureSet1D/2D of
    device tensors (east, eps re-derived from the stored records exactly as
    every kernel does: ceil, offset, the eps >= 1 guard, wrap)."""

    def __init__(self, level: Level):
        self.level = level

    def __len__(self):
        return int(self.level.s_x.shape[0])

    @staticmethod
    def _dec(s: torch.Tensor, n: int):
        ef = torch.ceil(s)
        eps = ef - s
        hi = eps >= 1.0
        east = torch.remainder(ef.to(torch.int64) - hi.to(torch.int64), n)
        return east, torch.where(hi, eps - 1.0, eps)

    def __getitem__(self, k: int):
        lv = self.level
        if not -len(self) <= k < len(self):
            raise IndexError(k)
        n = lv.grid.n_x
        ex, epx = self._dec(lv.s_x[k], n)
        dx = lv.disp_x[k] if lv.disp_x is not None else None
        dt, t0 = lv.dt, (0.0 if lv.shared else k * lv.dt)
        if lv.grid.dim == 1:
            return DepartureSet1D(t0, dt, ex, epx, dx)
        ey, epy = self._dec(lv.s_y[k], n)
        dy = lv.disp_y[k] if lv.disp_y is not None else None
        return DepartureSet2D(t0, dt, ex, ey, epx, epy, dx, dy)

    def __iter__(self):
        return (self[k] for k in range(len(self)))


class SigmaView:
    """Read-only sequence of a level's correction fields (device vectors)."""

    def __init__(self, level: Level):
        self.level = level

    def __len__(self):
        return int(self.level.sig_x.shape[0])

    def __getitem__(self, k: int):
        lv = self.level
        if not -len(self) <= k < len(self):
            raise IndexError(k)
        return CorrectionField(lv.sig_x[k], None if lv.sig_y is None else lv.sig_y[k])

    def __iter__(self):
        return (self[k] for k in range(len(self)))


def stencil_tables(level: Level):
    """The 1D gather tables of Level._ensure_stencils (mgrit.py:121-126):
    idx (S, n_x, p+1) int32 = (east + offsets) mod n_x and the weights."""
    if level.grid.dim != 1 or level.s_x is None:
        return None, None
    ell, r = stencil_extents(level.p)
    deps = DepartureSetView(level)
    n = level.grid.n_x
    offs = torch.arange(-ell, r + 1, device=level.s_x.device)
    idx, w = [], []
    for d in deps:
        idx.append(torch.remainder(d.east[:, None] + offs[None, :], n).to(torch.int32))
        w.append(interp_weights(level.p, d.eps))
    return torch.stack(idx), torch.stack(w)
