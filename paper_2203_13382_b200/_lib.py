"""ctypes binding of libmgrit_b200.so (include/mgrit_b200.h).

The product path has no CPU fallback: importing the operators without the
built library, or calling them without a CUDA device, raises immediately.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_lib", "libmgrit_b200.so")

MGRIT_OK, MGRIT_EINVAL, MGRIT_ECUDA = 0, 2, 3
KIND_SL, KIND_CORRECTED, KIND_FORWARD_EULER = 0, 1, 2
PHASE_FC, PHASE_F_RES, PHASE_FONLY_RES, PHASE_INJ_F = 0, 1, 2, 3
SPEED_IDS = {"C1": 1, "C2": 2, "C3": 3, "C4": 4, "C5": 5, "B2": 6, "B4": 7}

c_i32, c_i64, c_u64, c_dbl, c_vp = ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64, ctypes.c_double, ctypes.c_void_p


class LevelDesc(ctypes.Structure):
    _fields_ = [
        ("dim", c_i32), ("n_x", c_i32), ("p", c_i32), ("kind", c_i32),
        ("shared", c_i32), ("n_steps", c_i32), ("n_points", c_i64),
        ("s_x", c_vp), ("s_y", c_vp), ("sig_x", c_vp), ("sig_y", c_vp),
        ("gmres_max_iters", c_i32), ("stencil_numba", c_i32), ("gmres_tol", c_dbl),
        ("gmres_lowsync", c_i32), ("launch_policy", c_i32),
        ("sl2d_separable", c_i32), ("pad_", c_i32),
    ]


class ErkTableau(ctypes.Structure):
    _fields_ = [("n_stages", c_i32), ("pad", c_i32), ("a", c_dbl * 36), ("b", c_dbl * 6), ("c", c_dbl * 6)]


class PhaseArgs(ctypes.Structure):
    _fields_ = [
        ("phase", c_i32), ("m", c_i32),
        ("c_begin", c_i64), ("c_count", c_i64), ("n_intervals", c_i64),
        ("U", c_vp), ("ldu", c_i64), ("u_row0", c_i64),
        ("G", c_vp), ("ldg", c_i64), ("g_row0", c_i64),
        ("Cbuf", c_vp), ("Uc", c_vp), ("Gc", c_vp), ("c_row0", c_i64),
        ("partial", c_vp), ("partial0", c_i64),
        ("zero_init", c_i32), ("f_relaxed", c_i32),
    ]


# name -> (restype, argtypes)
_SIGS = {
    "mgrit_abi_version": (ctypes.c_int, []),
    "mgrit_last_error": (ctypes.c_char_p, []),
    "mgrit_gmres_scratch_bytes": (c_i64, [ctypes.POINTER(LevelDesc), c_i64]),
    "mgrit_resident_rows": (c_i64, [ctypes.POINTER(LevelDesc)]),
    "mgrit_erk_departures": (ctypes.c_int, [c_i32, c_i32, c_i32, ctypes.POINTER(ErkTableau), c_i64, c_i64,
                                            c_dbl, c_i32, c_dbl, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "mgrit_departures_from_coords": (ctypes.c_int, [c_i32, c_i32, c_i64, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "mgrit_backtrack": (ctypes.c_int, [c_i32, c_i32, c_i32, c_i64, c_i32, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "mgrit_phi_sigma": (ctypes.c_int, [c_i32, c_i32, c_i32, c_i32, c_i64, c_i32, c_vp, c_vp, c_vp, c_vp, c_vp,
                                       c_vp, c_vp, c_vp, c_vp]),
    "mgrit_records_separable": (ctypes.c_int, [c_i32, c_i64, c_vp, c_vp, c_vp, c_vp]),
    "mgrit_pcg64_fill": (ctypes.c_int, [c_u64, c_u64, c_u64, c_u64, c_i64, c_i32, c_vp, c_vp]),
    "mgrit_apply_rows": (ctypes.c_int, [ctypes.POINTER(LevelDesc), c_i64, c_vp, c_i64, c_i64, c_vp, c_i64,
                                        c_vp, c_i64, c_vp, c_i64, c_vp, c_i64, c_vp, c_vp, c_vp, c_i64,
                                        c_vp, c_vp]),
    "mgrit_level_phase": (ctypes.c_int, [ctypes.POINTER(LevelDesc), ctypes.POINTER(PhaseArgs), c_vp, c_i64,
                                         c_vp, c_vp]),
    "mgrit_sequential_sweep": (ctypes.c_int, [ctypes.POINTER(LevelDesc), c_vp, c_i64, c_vp, c_i64, c_i32,
                                              c_vp, c_vp, c_i64, c_vp, c_vp]),
    "mgrit_sum": (ctypes.c_int, [c_vp, c_i64, c_vp, c_vp]),
    "mgrit_axpy_rows": (ctypes.c_int, [c_vp, c_i64, c_i64, c_vp, c_i64, c_i64, c_i64, c_vp]),
    "mgrit_loop_begin": (ctypes.c_int, [c_vp, ctypes.POINTER(c_vp)]),
    "mgrit_loop_check": (ctypes.c_int, [c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "mgrit_loop_end": (ctypes.c_int, [c_vp, c_vp]),
    "mgrit_loop_init": (ctypes.c_int, [c_vp, c_vp, c_vp, c_vp, c_dbl, c_dbl, c_i32, c_vp]),
    "mgrit_loop_launch": (ctypes.c_int, [c_vp, c_vp]),
    "mgrit_loop_destroy": (None, [c_vp]),
    "mgrit_loop_body_kernels": (c_i64, [c_vp]),
    "mgrit_decompose": (ctypes.c_int, [c_i32, c_i64, c_vp, c_vp, c_vp, c_vp]),
    "mgrit_interp_weights": (ctypes.c_int, [c_i32, c_i64, c_vp, c_vp, c_vp]),
    "mgrit_records_from_east_eps": (ctypes.c_int, [c_i32, c_i64, c_vp, c_vp, c_vp, c_vp]),
    "mgrit_apply_imsd": (ctypes.c_int, [c_i32, c_i32, c_i32, c_i64, c_vp, c_vp, c_vp, c_i64, c_vp, c_i64, c_vp]),
    "mgrit_apply_rows_hist": (ctypes.c_int, [ctypes.POINTER(LevelDesc), c_i64, c_vp, c_i64, c_i64, c_vp, c_i64,
                                             c_vp, c_i64, c_vp, c_vp, c_vp, c_i64, c_vp, c_vp]),
}

LOOP_STATES = {0: "running", 1: "converged", 2: "diverged", 3: "max_iters"}

EXPORTED = tuple(_SIGS)

_LIB = None


def load(path: str | None = None):
    """Load the shared library (no CUDA context needed)."""
    global _LIB
    if _LIB is not None and path is None:
        return _LIB
    p = path or LIB_PATH
    if not os.path.exists(p):
        raise RuntimeError(
            f"libmgrit_b200.so not built ({p}); run `python -m paper_2203_13382_b200._build` "
            "(there is no CPU fallback)")
    lib = ctypes.CDLL(p)
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.mgrit_abi_version() != 3:
        raise RuntimeError("libmgrit_b200.so ABI mismatch")
    if path is None:
        _LIB = lib
    return lib


def check(rc: int, what: str):
    if rc != MGRIT_OK:
        msg = _LIB.mgrit_last_error().decode() if _LIB is not None else ""
        kind = "invalid argument" if rc == MGRIT_EINVAL else "CUDA error"
        raise RuntimeError(f"{what}: {kind} ({rc}) {msg}")


def erk_tableau(order: int) -> ErkTableau:
    """The reference's ERK tableaux (semi_lagrangian.py:46-72), same constants."""
    if order == 1:
        a = np.zeros((1, 1)); b = np.array([1.0]); c = np.array([0.0])
    elif order == 3:
        a = np.array([[0.0, 0.0, 0.0], [0.5, 0.0, 0.0], [-1.0, 2.0, 0.0]])
        b = np.array([1.0 / 6.0, 2.0 / 3.0, 1.0 / 6.0])
        c = np.array([0.0, 0.5, 1.0])
    elif order == 5:
        a = np.zeros((6, 6))
        a[1, 0] = 1.0 / 4.0
        a[2, :2] = [3.0 / 32.0, 9.0 / 32.0]
        a[3, :3] = [1932.0 / 2197.0, -7200.0 / 2197.0, 7296.0 / 2197.0]
        a[4, :4] = [439.0 / 216.0, -8.0, 3680.0 / 513.0, -845.0 / 4104.0]
        a[5, :5] = [-8.0 / 27.0, 2.0, -3544.0 / 2565.0, 1859.0 / 4104.0, -11.0 / 40.0]
        b = np.array([16.0 / 135.0, 0.0, 6656.0 / 12825.0, 28561.0 / 56430.0, -9.0 / 50.0, 2.0 / 55.0])
        c = np.array([0.0, 1.0 / 4.0, 3.0 / 8.0, 12.0 / 13.0, 1.0, 0.5])
    else:
        raise ValueError(f"unsupported ERK order {order}; supported: 1, 3, 5")
    t = ErkTableau()
    t.n_stages = len(b)
    full = np.zeros((6, 6))
    full[: a.shape[0], : a.shape[1]] = a
    for i in range(36):
        t.a[i] = float(full.ravel()[i])
    for i in range(len(b)):
        t.b[i] = float(b[i])
        t.c[i] = float(c[i])
    return t
