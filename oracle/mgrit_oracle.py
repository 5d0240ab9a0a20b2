"""CPU restatement of the reference MGRIT semi-Lagrangian solver (TEST ORACLE).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's CPU legs.  Never shipped on the product path.

Every function cites the reference location (relative to
/root/reference/pkg/src/mgrit_advect/) whose arithmetic it restates.  The
floating-point operation order follows the reference so that:

* the plain SL gather (``sl_apply``) is bit-identical to ``Level.step_batch``
  / ``sl_step`` (strict left-to-right sum of separately rounded products);
* ERK tracing, decomposition, backtracking and phi/sigma reproduce the
  reference bit-for-bit on the same numpy build;
* GMRES uses the same numpy/BLAS calls (dot, norm, solve, matmul) as
  ``gmres_solve`` and the C sweep (``sweep.c``) uses the same sequential loops
  as the numba kernel.

Extensions over the reference, needed by BASELINE.json's configs (SURVEY.md
Appendix A): wave speeds ``B2`` (1+0.5 sin(2 pi x) cos(2 pi t)) and ``B4``
((cos^2(pi x) cos(2 pi t) + 0.5, sin^2(pi y) cos(2 pi t) + 0.5)), the ``sin4``
initial state and the ``pm1`` (uniform [-1, 1)) initial iterate.
"""

from __future__ import annotations

import ctypes
import math
import os
import time
from dataclasses import dataclass, field
from typing import Callable, Sequence

import numpy as np

__all__ = [
    "SPEEDS", "speed_is_constant", "speed_dim", "eval_speed",
    "nodes", "erk_tableau", "erk_trace", "decompose", "lagrange_weights",
    "Departures", "departures_from_coords", "erk_departures", "sl_apply",
    "f_poly", "d_stencil", "circulant", "imsd", "phi_sigma", "gmres",
    "backtrack", "OLevel", "OConfig", "hierarchy", "f_relax", "c_relax",
    "residual", "solve_sequential", "v_cycle", "solve", "sequential",
    "initial_state", "initial_iterate", "st_norm", "sweep_available", "GmresLog", "OReport",
]

TWO_PI = 2.0 * np.pi

# ---------------------------------------------------------------------------
# wave speeds: core.py:130-153 (catalog C1..C5) + BASELINE.json speeds B2/B4.
# Each entry: (dim, constant, tuple of component closures).


def _ones(a):
    return np.ones_like(np.asarray(a, dtype=float))


SPEEDS: dict[str, tuple[int, bool, tuple[Callable, ...]]] = {
    "C1": (1, True, (lambda x, t: _ones(x),)),
    "C2": (1, False, (lambda x, t: np.cos(TWO_PI * t) * _ones(x),)),
    "C3": (1, False, (lambda x, t: np.cos(TWO_PI * t) * np.cos(TWO_PI * x),)),
    "C4": (2, True, (lambda x, y, t: _ones(x), lambda x, y, t: _ones(y))),
    "C5": (2, False, (
        lambda x, y, t: np.sin(np.pi * y) ** 2 * np.cos(TWO_PI * t / 3.4),
        lambda x, y, t: -np.cos(np.pi * x) ** 2 * np.cos(TWO_PI * t / 3.4),
    )),
    # BASELINE.json configs 2-3 (advective form)
    "B2": (1, False, (lambda x, t: 1.0 + 0.5 * np.sin(TWO_PI * x) * np.cos(TWO_PI * t),)),
    # BASELINE.json configs 4-5
    "B4": (2, False, (
        lambda x, y, t: np.cos(np.pi * x) ** 2 * np.cos(TWO_PI * t) + 0.5,
        lambda x, y, t: np.sin(np.pi * y) ** 2 * np.cos(TWO_PI * t) + 0.5,
    )),
}


def speed_dim(name: str) -> int:
    return SPEEDS[name][0]


def speed_is_constant(name: str) -> bool:
    return SPEEDS[name][1]


def eval_speed(name: str, comp: int, *args):
    return SPEEDS[name][2][comp](*args)


# ---------------------------------------------------------------------------
# grids: core.py:17-82 (x_lo=-1, length=2, nodes x_lo + h*i, 2D flat x fastest)


def nodes(dim: int, n_x: int):
    h = 2.0 / n_x
    x1 = -1.0 + h * np.arange(n_x)
    if dim == 1:
        return x1
    return np.tile(x1, n_x), np.repeat(x1, n_x)


# ---------------------------------------------------------------------------
# ERK tableaux: semi_lagrangian.py:46-72


def erk_tableau(order: int):
    if order == 1:
        return np.zeros((1, 1)), np.array([1.0]), np.array([0.0])
    if order == 3:
        return (np.array([[0.0, 0.0, 0.0], [0.5, 0.0, 0.0], [-1.0, 2.0, 0.0]]),
                np.array([1.0 / 6.0, 2.0 / 3.0, 1.0 / 6.0]), np.array([0.0, 0.5, 1.0]))
    if order == 5:
        a = np.zeros((6, 6))
        a[1, 0] = 1.0 / 4.0
        a[2, :2] = [3.0 / 32.0, 9.0 / 32.0]
        a[3, :3] = [1932.0 / 2197.0, -7200.0 / 2197.0, 7296.0 / 2197.0]
        a[4, :4] = [439.0 / 216.0, -8.0, 3680.0 / 513.0, -845.0 / 4104.0]
        a[5, :5] = [-8.0 / 27.0, 2.0, -3544.0 / 2565.0, 1859.0 / 4104.0, -11.0 / 40.0]
        b = np.array([16.0 / 135.0, 0.0, 6656.0 / 12825.0, 28561.0 / 56430.0, -9.0 / 50.0, 2.0 / 55.0])
        c = np.array([0.0, 1.0 / 4.0, 3.0 / 8.0, 12.0 / 13.0, 1.0, 0.5])
        return a, b, c
    raise ValueError(f"unsupported ERK order {order}")


def erk_trace(speed: str, arrival, t_start: float, dt: float, order: int):
    """One backward ERK step of size -dt from t_start+dt (semi_lagrangian.py:75-115).

    Stage sums add (hs*a_sj)*k_j only for non-zero a_sj; the final sum adds
    (hs*b_s)*k_s for every stage, in stage order.
    """
    a, b, c = erk_tableau(order)
    hs = -dt
    t1 = t_start + dt
    dim = speed_dim(speed)
    pts = [np.asarray(arrival, dtype=float)] if dim == 1 else [np.asarray(v, dtype=float) for v in arrival]
    ks: list[list[np.ndarray]] = [[] for _ in range(dim)]
    for s in range(len(b)):
        stage = [p.copy() for p in pts]
        for j in range(s):
            if a[s, j] != 0.0:
                coef = hs * a[s, j]
                stage = [stage[d] + coef * ks[d][j] for d in range(dim)]
        ts = t1 + c[s] * hs
        for d in range(dim):
            ks[d].append(eval_speed(speed, d, *stage, ts))
    out = [p.copy() for p in pts]
    for s in range(len(b)):
        coef = hs * b[s]
        out = [out[d] + coef * ks[d][s] for d in range(dim)]
    return out[0] if dim == 1 else (out[0], out[1])


# ---------------------------------------------------------------------------
# decomposition + weights: semi_lagrangian.py:118-161


def decompose(n_x: int, coords):
    """(east index mod n_x, eps in [0,1)) with the reference's rounding guards."""
    h = 2.0 / n_x
    s = np.mod(np.asarray(coords, dtype=float) - (-1.0), 2.0) / h
    ef = np.ceil(s)
    eps = ef - s
    east = ef.astype(np.int64)
    eps = np.where(eps < 0.0, 0.0, eps)
    hi = eps >= 1.0
    eps = np.where(hi, eps - 1.0, eps)
    east = np.where(hi, east - 1, east)
    return np.mod(east, n_x), eps


def extents(p: int):
    if p not in (1, 3, 5):
        raise ValueError(f"unsupported interpolation degree p={p}")
    return (p + 1) // 2, (p - 1) // 2


def lagrange_weights(p: int, eps):
    """w[:, j] = prod_{q != j} (z - q) / prod_{q != j} (j - q), z = -eps."""
    ell, r = extents(p)
    z = -np.atleast_1d(np.asarray(eps, dtype=float))
    offs = list(range(-ell, r + 1))
    w = np.empty((z.shape[0], p + 1))
    for col, j in enumerate(offs):
        num = np.ones_like(z)
        den = 1.0
        for q in offs:
            if q != j:
                num = num * (z - q)
                den *= j - q
        w[:, col] = num / den
    return w


@dataclass
class Departures:
    """One step's departure record (DepartureSet1D/2D, semi_lagrangian.py:164-205).

    ``coords`` keeps the traced departure coordinates (tuple in 2D) so the GPU
    side can be fed exactly the same record.
    """

    east: tuple          # (east_x,) or (east_x, east_y)
    eps: tuple           # (eps,) or (eps, nu)
    disp: tuple          # arrival - departure per axis
    coords: tuple


def departures_from_coords(dim: int, n_x: int, coords) -> Departures:
    if dim == 1:
        cx = (np.asarray(coords, dtype=float),)
        arr = (nodes(1, n_x),)
    else:
        cx = tuple(np.asarray(c, dtype=float) for c in coords)
        arr = nodes(2, n_x)
    east, eps, disp = [], [], []
    for d in range(dim):
        e, x = decompose(n_x, cx[d])
        east.append(e)
        eps.append(x)
        disp.append(arr[d] - cx[d])
    return Departures(tuple(east), tuple(eps), tuple(disp), cx)


def erk_departures(dim, n_x, speed, t_start, dt, order) -> Departures:
    """semi_lagrangian.py:208-217."""
    arr = nodes(dim, n_x)
    return departures_from_coords(dim, n_x, erk_trace(speed, arr, t_start, dt, order))


def sl_apply(dim: int, n_x: int, p: int, dep: Departures, u: np.ndarray) -> np.ndarray:
    """One SL step (semi_lagrangian.py:220-253, mgrit.py:128-133, 152-166).

    1D: sum_j w_j u[(E+j) mod n], strictly left to right (the numpy reduction
    order of ``(u[idx]*w).sum(axis=1)``).  2D: x inner, y outer, from zero.
    Works on a single state (n,) or a batch (B, n) sharing one record.
    """
    ell, r = extents(p)
    offs = range(-ell, r + 1)
    if dim == 1:
        w = lagrange_weights(p, dep.eps[0])
        idx = [np.mod(dep.east[0] + j, n_x) for j in offs]
        acc = u[..., idx[0]] * w[:, 0]
        for col in range(1, p + 1):
            acc = acc + u[..., idx[col]] * w[:, col]
        return acc
    wx = lagrange_weights(p, dep.eps[0])
    wy = lagrange_weights(p, dep.eps[1])
    cols = [np.mod(dep.east[0] + j, n_x) for j in offs]
    rows = [np.mod(dep.east[1] + j, n_x) * n_x for j in offs]
    out = np.zeros(u.shape)
    for jy in range(p + 1):
        acc = np.zeros(u.shape)
        for jx in range(p + 1):
            acc += wx[:, jx] * u[..., rows[jy] + cols[jx]]
        out += wy[:, jy] * acc
    return out


# ---------------------------------------------------------------------------
# truncation-error correction: coarse_correction.py:22-56, 92-154


def f_poly(p: int, z):
    """prod_{q=-l}^{r} (q + z) / (p+1)!   (coarse_correction.py:22-32)."""
    ell, r = extents(p)
    z = np.asarray(z, dtype=float)
    out = np.ones_like(z)
    for q in range(-ell, r + 1):
        out = out * (q + z)
    return out / math.factorial(p + 1)


def d_stencil(p: int) -> np.ndarray:
    """Centred (p+1)st-difference integer stencil (coarse_correction.py:35-47)."""
    return {1: np.array([1.0, -2.0, 1.0]),
            3: np.array([1.0, -4.0, 6.0, -4.0, 1.0]),
            5: np.array([1.0, -6.0, 15.0, -20.0, 15.0, -6.0, 1.0])}[p]


def circulant(c: np.ndarray, v: np.ndarray) -> np.ndarray:
    """out = c0 v; out += (c_{+k} v_{i+k} + c_{-k} v_{i-k})  (coarse_correction.py:50-56)."""
    rad = (len(c) - 1) // 2
    out = c[rad] * v
    for k in range(1, rad + 1):
        out += c[rad + k] * np.roll(v, -k) + c[rad - k] * np.roll(v, k)
    return out


def imsd(sig: tuple, c: np.ndarray, v: np.ndarray, n_x: int) -> np.ndarray:
    """(I - diag(sigma) D) v, 1D or separable 2D (coarse_correction.py:130-149)."""
    if len(sig) == 1:
        return v - sig[0] * circulant(c, v)
    v2 = v.reshape(n_x, n_x)
    rad = (len(c) - 1) // 2
    dx = c[rad] * v2
    dy = c[rad] * v2
    for k in range(1, rad + 1):
        dx = dx + c[rad + k] * np.roll(v2, -k, axis=1) + c[rad - k] * np.roll(v2, k, axis=1)
        dy = dy + c[rad + k] * np.roll(v2, -k, axis=0) + c[rad - k] * np.roll(v2, k, axis=0)
    return v - sig[0] * dx.ravel() - sig[1] * dy.ravel()


def ipsd(sig, c, v, n_x):
    """Explicit factor I + diag(sigma) D = 2v - (I - diag(sigma)D)v (coarse_correction.py:152-154)."""
    return 2.0 * v - imsd(sig, c, v, n_x)


def phi_sigma(p: int, coarse: Departures, children: Sequence[Departures],
              child_sigma: Sequence[tuple] | None) -> tuple:
    """phi = (-1)^(p+1) (f(eps_c) - sum_k f(eps_k)) per axis, plus the children's
    sigma in order (coarse_correction.py:92-127, mgrit.py:249-256)."""
    sign = (-1.0) ** (p + 1)
    out = []
    for d in range(len(coarse.eps)):
        acc = f_poly(p, coarse.eps[d]).copy()
        for ch in children:
            acc -= f_poly(p, ch.eps[d])
        out.append(sign * acc)
    if child_sigma is not None:
        for cs in child_sigma:
            out = [out[d] + cs[d] for d in range(len(out))]
    return tuple(out)


class GmresLog:
    """Optional per-call GMRES iteration counter (for parity of counts)."""

    def __init__(self):
        self.counts: list[int] = []


def gmres(op: Callable[[np.ndarray], np.ndarray], rhs: np.ndarray, max_iters: int,
          tol: float | None, log: GmresLog | None = None):
    """Non-restarted MGS-GMRES, zero start, Givens (coarse_correction.py:173-228)."""
    if not np.all(np.isfinite(rhs)):
        raise ValueError("non-finite right-hand side in gmres")
    beta = np.linalg.norm(rhs)
    if beta == 0.0:
        if log is not None:
            log.counts.append(0)
        return np.zeros_like(rhs), np.array([0.0])
    n = rhs.shape[0]
    V = np.empty((max_iters + 1, n))
    H = np.zeros((max_iters + 1, max_iters))
    cs = np.zeros(max_iters)
    sn = np.zeros(max_iters)
    g = np.zeros(max_iters + 1)
    g[0] = beta
    V[0] = rhs / beta
    hist = [beta]
    done = 0
    for k in range(max_iters):
        w = np.array(op(V[k]), dtype=float)
        for j in range(k + 1):
            H[j, k] = np.dot(V[j], w)
            w -= H[j, k] * V[j]
        H[k + 1, k] = np.linalg.norm(w)
        brk = H[k + 1, k] <= 1e-14 * beta
        if not brk:
            V[k + 1] = w / H[k + 1, k]
        for j in range(k):
            t = cs[j] * H[j, k] + sn[j] * H[j + 1, k]
            H[j + 1, k] = -sn[j] * H[j, k] + cs[j] * H[j + 1, k]
            H[j, k] = t
        den = np.hypot(H[k, k], H[k + 1, k])
        cs[k] = H[k, k] / den
        sn[k] = H[k + 1, k] / den
        H[k, k] = den
        H[k + 1, k] = 0.0
        g[k + 1] = -sn[k] * g[k]
        g[k] = cs[k] * g[k]
        hist.append(abs(g[k + 1]))
        done = k + 1
        if brk or (tol is not None and hist[-1] <= tol * beta):
            break
    y = np.linalg.solve(np.triu(H[:done, :done]), g[:done])
    if log is not None:
        log.counts.append(done)
    return V[:done].T @ y, np.array(hist)


# ---------------------------------------------------------------------------
# backtracking: backtracking.py:21-86


def backtrack(dim: int, n_x: int, children: Sequence[Departures]) -> Departures:
    m = len(children)
    if dim == 1:
        x = nodes(1, n_x)
        c = x - children[m - 1].disp[0]
        for k in range(m - 2, -1, -1):
            d = children[k].disp[0]
            e, eps = decompose(n_x, c)
            west = np.mod(e - 1, n_x)
            c = c - ((1.0 - eps) * d[e] + eps * d[west])
        return departures_from_coords(1, n_x, c)
    x, y = nodes(2, n_x)
    cx = x - children[m - 1].disp[0]
    cy = y - children[m - 1].disp[1]
    for k in range(m - 2, -1, -1):
        dx, dy = children[k].disp
        e, eps = decompose(n_x, cx)
        nn, nu = decompose(n_x, cy)
        w_ = np.mod(e - 1, n_x)
        s_ = np.mod(nn - 1, n_x)
        ne, nw, se, sw = nn * n_x + e, nn * n_x + w_, s_ * n_x + e, s_ * n_x + w_
        a_ne = (1.0 - eps) * (1.0 - nu)
        a_nw = eps * (1.0 - nu)
        a_se = (1.0 - eps) * nu
        a_sw = eps * nu
        cx = cx - (a_ne * dx[ne] + a_nw * dx[nw] + a_se * dx[se] + a_sw * dx[sw])
        cy = cy - (a_ne * dy[ne] + a_nw * dy[nw] + a_se * dy[se] + a_sw * dy[sw])
    return departures_from_coords(2, n_x, (cx, cy))


# ---------------------------------------------------------------------------
# the C restatement of the numba sweep (sweep.c <- _kernels.py:18-131)

_SWEEP = None


def _sweep_lib():
    global _SWEEP
    if _SWEEP is None:
        here = os.path.dirname(os.path.abspath(__file__))
        path = os.path.join(here, "_build", "liboracle_sweep.so")
        if not os.path.exists(path):
            _SWEEP = False
        else:
            lib = ctypes.CDLL(path)
            P = ctypes.c_void_p
            lib.oracle_sequential_corrected_sweep.argtypes = [
                P, P, P, P, ctypes.c_int, P, P, ctypes.c_long, ctypes.c_long,
                ctypes.c_int, ctypes.c_double, ctypes.c_int, ctypes.c_int, P]
            lib.oracle_sequential_corrected_sweep.restype = None
            _SWEEP = lib
    return _SWEEP or None


def sweep_available() -> bool:
    return _sweep_lib() is not None


# ---------------------------------------------------------------------------
# levels and hierarchy: mgrit.py:39-269


@dataclass
class OConfig:
    """SolverConfig (mgrit.py:39-86) plus BASELINE extensions (u0, iterate)."""

    n_x: int
    n_t: int
    dim: int = 1
    wave_speed: str = "C1"
    p: int = 1
    r: int | None = None
    dt: float | None = None
    schedule: int | Sequence[int] = 4
    max_levels: int | None = None
    operator_kind: str = "corrected"
    departure_policy: str = "backtrack"
    gmres_mode: str | None = None
    relaxation: str = "FCF"
    seed: int = 0
    rtol: float = 1e-10
    max_iters: int = 100
    divergence_factor: float = 1e6
    u0: str = "reference"          # "reference" (core.py:164-170) | "sin4" (BASELINE)
    iterate: str = "uniform01"     # "uniform01" (mgrit.py:353) | "pm1" (BASELINE cfg 1)

    def factor(self, li: int) -> int:
        if isinstance(self.schedule, int):
            return self.schedule
        seq = list(self.schedule)
        return seq[min(li, len(seq) - 1)]

    @property
    def order(self) -> int:
        return self.p if self.r is None else self.r


@dataclass
class OLevel:
    index: int
    dim: int
    n_x: int
    p: int
    n_steps: int
    dt: float
    kind: str
    deps: list | None
    sigma: list | None = None
    gmres: tuple | None = None       # (max_iters, tol or None)
    cf: int | None = None
    finer: "OLevel | None" = None
    shared: bool = False
    log: GmresLog | None = field(default=None, repr=False)

    @property
    def n_points(self) -> int:
        return self.n_x ** self.dim

    def dep(self, n):
        return self.deps[0] if self.shared else self.deps[n]

    def sig(self, n):
        return self.sigma[0] if self.shared else self.sigma[n]

    def step(self, n: int, u: np.ndarray) -> np.ndarray:
        """mgrit.py:135-150."""
        if self.kind == "ideal":
            ratio = self.finer.n_steps // self.n_steps
            for k in range(ratio):
                u = self.finer.step(n * ratio + k, u)
            return u
        v = sl_apply(self.dim, self.n_x, self.p, self.dep(n), u)
        if self.kind == "corrected":
            c = d_stencil(self.p)
            s = self.sig(n)
            v, _ = gmres(lambda w: imsd(s, c, w, self.n_x), v, self.gmres[0], self.gmres[1], self.log)
        elif self.kind == "forward_euler":
            v = ipsd(self.sig(n), d_stencil(self.p), v, self.n_x)
        return v

    def step_batch(self, t_idx, U: np.ndarray) -> np.ndarray:
        """mgrit.py:152-167: vectorised plain SL for 1D, row loop otherwise."""
        if self.dim == 1 and self.kind in ("fine", "rediscretized"):
            if self.shared:
                return sl_apply(1, self.n_x, self.p, self.deps[0], U)
            return np.stack([sl_apply(1, self.n_x, self.p, self.deps[int(t)], u)
                             for t, u in zip(t_idx, U)]) if len(t_idx) else np.empty_like(U)
        return np.stack([self.step(int(t), u) for t, u in zip(t_idx, U)])


def hierarchy(cfg: OConfig) -> list[OLevel]:
    """build_hierarchy (mgrit.py:217-269) with the backtrack / erk_rediscretized /
    erk_substeps departure policies (mgrit.py:185-214)."""
    dim, n_x = cfg.dim, cfg.n_x
    if speed_dim(cfg.wave_speed) != dim:
        raise ValueError("wave speed dimension does not match config")
    h = 2.0 / n_x
    dt = cfg.dt if cfg.dt is not None else 0.85 * h
    order = cfg.order
    shared = speed_is_constant(cfg.wave_speed)
    count = 1 if shared else cfg.n_t
    fine_deps = [erk_departures(dim, n_x, cfg.wave_speed, n * dt, dt, order) for n in range(count)]
    levels = [OLevel(0, dim, n_x, cfg.p, cfg.n_t, dt, "fine", fine_deps, shared=shared)]
    while True:
        if cfg.max_levels is not None and len(levels) >= cfg.max_levels:
            break
        prev = levels[-1]
        m = cfg.factor(len(levels) - 1)
        if prev.n_steps % m != 0 or prev.n_steps // m < 2:
            break
        n_c = prev.n_steps // m
        dt_c = prev.dt * m
        if cfg.operator_kind == "ideal":
            lvl = OLevel(len(levels), dim, n_x, cfg.p, n_c, dt_c, "ideal", None, finer=prev)
        else:
            deps = []
            for n in range(1 if shared else n_c):
                t0 = n * dt_c
                if cfg.departure_policy == "backtrack":
                    deps.append(backtrack(dim, n_x, [prev.dep(n * m + k) for k in range(m)]))
                elif cfg.departure_policy == "erk_rediscretized":
                    deps.append(erk_departures(dim, n_x, cfg.wave_speed, t0, dt_c, order))
                else:
                    n_sub = int(round(dt_c / dt))
                    arr = nodes(dim, n_x)
                    c = arr
                    for k in range(n_sub - 1, -1, -1):
                        c = erk_trace(cfg.wave_speed, c, t0 + k * dt, dt, order)
                    deps.append(departures_from_coords(dim, n_x, c))
            sigma = None
            if cfg.operator_kind in ("corrected", "forward_euler"):
                sigma = []
                for n in range(1 if shared else n_c):
                    ch = [prev.dep(n * m + k) for k in range(m)]
                    chs = [prev.sig(n * m + k) for k in range(m)] if prev.sigma is not None else None
                    sigma.append(phi_sigma(cfg.p, deps[n], ch, chs))
            lvl = OLevel(len(levels), dim, n_x, cfg.p, n_c, dt_c, cfg.operator_kind, deps, sigma,
                         finer=prev, shared=shared)
        prev.cf = m
        levels.append(lvl)
    if len(levels) < 2:
        raise ValueError("time grid does not admit any coarsening with the given schedule")
    mode = cfg.gmres_mode or ("fixed" if len(levels) == 2 else "tolerance")
    gm = (10, None) if mode == "fixed" else (10, 1e-2)
    for lvl in levels[1:]:
        lvl.gmres = gm
    return levels


# ---------------------------------------------------------------------------
# relaxation / residual / cycle / solve: mgrit.py:276-390


def f_relax(lev: OLevel, U, G, m=None):
    m = lev.cf if m is None else m
    starts = np.arange(0, lev.n_steps, m)
    for k in range(1, m):
        t = starts + k - 1
        U[t + 1] = lev.step_batch(t, U[t]) + G[t + 1]


def c_relax(lev: OLevel, U, G, m=None):
    m = lev.cf if m is None else m
    t = np.arange(m, lev.n_steps + 1, m) - 1
    U[t + 1] = lev.step_batch(t, U[t]) + G[t + 1]


def residual(lev: OLevel, U, G):
    R = np.empty_like(U)
    R[0] = 0.0
    t = np.arange(lev.n_steps)
    R[1:] = G[1:] + lev.step_batch(t, U[:-1]) - U[1:]
    return R


def solve_sequential(lev: OLevel, U, G):
    """mgrit.py:302-314: the native sweep for 1D corrected levels with >= 64 steps."""
    lib = _sweep_lib()
    if lib is not None and lev.dim == 1 and lev.kind == "corrected" and lev.n_steps >= 64:
        n = lev.n_x
        ell, r = extents(lev.p)
        S = len(lev.deps)
        idx = np.stack([np.stack([np.mod(d.east[0] + j, n) for j in range(-ell, r + 1)], axis=1)
                        for d in lev.deps]).astype(np.int32)
        w = np.stack([lagrange_weights(lev.p, d.eps[0]) for d in lev.deps])
        sig = np.ascontiguousarray(np.stack([s[0] for s in lev.sigma]))
        c = d_stencil(lev.p)
        assert U.flags.c_contiguous and G.flags.c_contiguous and U.dtype == np.float64
        idx = np.ascontiguousarray(idx)
        w = np.ascontiguousarray(w)
        counts = np.zeros(lev.n_steps, dtype=np.int32)
        tol = -1.0 if lev.gmres[1] is None else lev.gmres[1]
        lib.oracle_sequential_corrected_sweep(
            idx.ctypes.data, w.ctypes.data, sig.ctypes.data, c.ctypes.data, len(c),
            U.ctypes.data, G.ctypes.data, U.shape[0] - 1, n, lev.p + 1, tol,
            lev.gmres[0], int(lev.shared), counts.ctypes.data)
        if lev.log is not None:
            lev.log.counts.extend(int(x) for x in counts)
        return
    for n in range(1, lev.n_steps + 1):
        U[n] = lev.step(n - 1, U[n - 1]) + G[n]


def v_cycle(levels, li, U, G, relaxation="FCF"):
    lev = levels[li]
    if li == len(levels) - 1:
        solve_sequential(lev, U, G)
        return
    m = lev.cf
    f_relax(lev, U, G)
    if relaxation == "FCF":
        c_relax(lev, U, G)
        f_relax(lev, U, G)
    R = residual(lev, U, G)
    Gc = R[::m].copy()
    Uc = np.zeros((lev.n_steps // m + 1, lev.n_points))
    v_cycle(levels, li + 1, Uc, Gc, relaxation)
    U[::m] += Uc
    f_relax(lev, U, G)


def st_norm(R) -> float:
    """core.py:173-181 (flat two-norm via BLAS)."""
    return float(np.linalg.norm(np.asarray(R).ravel()))


def initial_state(cfg: OConfig) -> np.ndarray:
    """core.py:164-170 ("reference") or BASELINE's sin^4 product ("sin4")."""
    if cfg.dim == 1:
        return np.sin(np.pi * nodes(1, cfg.n_x)) ** 4
    x, y = nodes(2, cfg.n_x)
    if cfg.u0 == "sin4":
        return np.sin(np.pi * x) ** 4 * np.sin(np.pi * y) ** 4
    return np.sin(0.5 * np.pi * (x - 1.0)) ** 2 * np.sin(0.5 * np.pi * (y - 1.0)) ** 2


def initial_iterate(cfg: OConfig) -> np.ndarray:
    """mgrit.py:350-353: PCG64(seed).random((n_t, n_points)); BASELINE cfg 1 maps to [-1,1)."""
    rng = np.random.default_rng(cfg.seed)
    X = rng.random((cfg.n_t, cfg.n_x ** cfg.dim))
    if cfg.iterate == "pm1":
        X = 2.0 * X - 1.0
    return X


@dataclass
class OReport:
    residual_norms: np.ndarray
    iterations: int
    status: str
    final_factor: float
    wall_time: float
    gmres_counts: list | None = None


def solve(cfg: OConfig, levels=None, on_iter: Callable | None = None, log_gmres=False, iterate0=None):
    """mgrit.py:337-378 with BASELINE's u0/iterate hooks and an optional
    per-iteration callback ``on_iter(k, U)`` for snapshots."""
    t0 = time.perf_counter()
    if levels is None:
        levels = hierarchy(cfg)
    log = GmresLog() if log_gmres else None
    for lv in levels:
        lv.log = log
    fine = levels[0]
    U = np.empty((cfg.n_t + 1, fine.n_points))
    U[0] = initial_state(cfg)
    U[1:] = initial_iterate(cfg) if iterate0 is None else iterate0
    G = np.zeros_like(U)
    r0 = st_norm(residual(fine, U, G))
    hist = [r0]
    status = "max_iters"
    for it in range(cfg.max_iters):
        try:
            v_cycle(levels, 0, U, G, cfg.relaxation)
            r = st_norm(residual(fine, U, G))
        except (ValueError, FloatingPointError):
            hist.append(float("nan"))
            status = "diverged"
            break
        hist.append(r)
        if on_iter is not None:
            on_iter(it + 1, U)
        if not np.isfinite(r) or r >= cfg.divergence_factor * r0:
            status = "diverged"
            break
        if r <= cfg.rtol * r0:
            status = "converged"
            break
    h = np.array(hist)
    fac = float(h[-1] / h[-2]) if len(h) > 1 else float("nan")
    rep = OReport(h, len(h) - 1, status, fac, time.perf_counter() - t0,
                  list(log.counts) if log is not None else None)
    return rep, U


def sequential(cfg: OConfig, levels=None) -> np.ndarray:
    """sequential_reference (mgrit.py:381-390)."""
    if levels is None:
        from dataclasses import replace
        levels = hierarchy(replace(cfg, max_levels=2))
    fine = levels[0]
    U = np.empty((cfg.n_t + 1, fine.n_points))
    U[0] = initial_state(cfg)
    G = np.zeros_like(U)
    solve_sequential(fine, U, G)
    return U
