"""Numpy restatement of the fused phase-kernel semantics (test infrastructure).

Mirrors paper_2203_13382_b200/csrc/step1d_kernels.cuh:phase_kernel and
sweep_kernel line by line, with the oracle's step operator (the reference's
arithmetic) in place of the CUDA one, so the time-parallel engine's sharding
and halo logic (paper_2203_13382_b200/timepar.py) can run over gloo on CPU.
"""

from __future__ import annotations

import numpy as np
import torch

FC, F_RES, FONLY_RES, INJ_F = 0, 1, 2, 3


class OraclePhaseBackend:
    def __init__(self, olevels):
        self.lv = olevels
        self.bad_flag = False

    def _step(self, li, t, v):
        try:
            return self.lv[li].step(t, v)
        except ValueError:
            self.bad_flag = True
            return np.full_like(v, np.nan)

    def phase(self, li, phase, *, m, c_begin, c_count, n_intervals, U, u_row0, G, g_row0, Cbuf, Uc, Gc,
              c_row0, partial, partial0, zero_init):
        U = U.numpy()
        G = None if G is None else G.numpy()
        Cb = Cbuf.numpy()
        Ucn = None if Uc is None else Uc.numpy()
        Gcn = None if Gc is None else Gc.numpy()
        par = None if partial is None else partial.numpy()
        n = U.shape[1]

        def g(t):
            return G[t - g_row0] if G is not None else 0.0

        for c in range(c_begin, c_begin + c_count):
            t0, tC = c * m, c * m + m
            if zero_init and (c == 0 or phase in (FC, FONLY_RES)):
                v = np.zeros(n)
                if c == 0 or phase == FONLY_RES:
                    U[t0 - u_row0] = v
            elif phase in (FC, FONLY_RES) or c == 0:
                v = U[t0 - u_row0].copy()
            else:
                v = Cb[c - c_row0].copy()
            if phase == INJ_F:
                v = v + Ucn[c - c_row0]
                U[t0 - u_row0] = v
            elif phase == F_RES and c > 0:
                U[t0 - u_row0] = v
            last = c + 1 == n_intervals
            kmax = m - 1 if (phase == INJ_F and par is None) else m
            if phase == INJ_F and par is None and last:
                U[tC - u_row0] = Cb[c + 1 - c_row0] + Ucn[c + 1 - c_row0]
            for k in range(1, kmax + 1):
                t = t0 + k
                S = self._step(li, t - 1, v)
                if k < m:
                    v = S + g(t)
                    U[t - u_row0] = v
                    continue
                if phase == FC:
                    Cb[c + 1 - c_row0] = S + g(tC)
                    break
                if phase == INJ_F:
                    right = Cb[c + 1 - c_row0] + Ucn[c + 1 - c_row0]
                    if last:
                        U[tC - u_row0] = right
                elif phase == F_RES:
                    right = Cb[c + 1 - c_row0].copy()
                    U[tC - u_row0] = right
                else:
                    if zero_init:
                        right = np.zeros(n)
                        U[tC - u_row0] = right
                    else:
                        right = U[tC - u_row0].copy()
                    Cb[c + 1 - c_row0] = right
                r = (g(tC) + S) - right
                if Gcn is not None and phase != INJ_F:
                    Gcn[c + 1 - c_row0] = r
                if par is not None:
                    par[c - partial0] = float(np.dot(r, r))

    def sweep(self, li, U, G, zero_init):
        U = U.numpy()
        G = None if G is None else G.numpy()
        if zero_init:
            U[0] = 0.0
        for t in range(self.lv[li].n_steps):
            U[t + 1] = self._step(li, t, U[t]) + (G[t + 1] if G is not None else 0.0)

    def total(self, x: torch.Tensor, out: torch.Tensor):
        xs = x.numpy()
        acc = 0.0
        for v in xs:          # fixed global order
            acc += float(v)
        out.fill_(acc)

    def bad(self):
        return self.bad_flag
