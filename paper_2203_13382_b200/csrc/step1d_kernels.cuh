// step1d_kernels.cuh — the 1D hot path: batched SL / corrected / forward-Euler step
// operators and the fused MGRIT level phases.
//
// Design (B200): a 1D state row (n <= 16384 fp64 = 128 KB) fits in one SM's
// shared memory, so a CTA owns a whole row.  The fused phase kernels give one
// CTA per C-interval and walk its m-1 dependent F-steps with the state kept
// in shared memory: per step only the departure record (8 B/node) is read
// and the new state (8 B/node) written to HBM; the previous state never
// round-trips through HBM.  The semi-Lagrangian gather reads the smem row;
// the corrected operator's GMRES runs inside the CTA (block reductions for
// the MGS dots, one elected thread for the Givens/Hessenberg recurrences)
// with its Krylov basis in a per-CTA global scratch slab that stays L2
// resident.  Grids are persistent (<= resident-CTA capacity), looping over
// rows / intervals.
#include "internal.cuh"

namespace mgrit {

constexpr int kMaxKrylov = 16;

// per-CTA GMRES control block in shared memory
struct GmresSmem {
    double H[(kMaxKrylov + 1) * kMaxKrylov];
    double cs[kMaxKrylov], sn[kMaxKrylov], g[kMaxKrylov + 1], y[kMaxKrylov];
    int stop, done;
};

struct RowCtx {
    double *rowbuf;   // smem, n doubles: state row / Krylov vector for the stencil
    double *red;      // smem, NT/32+1 doubles
    GmresSmem *gs;    // smem
    double *basis;    // global, (K+1)*n doubles (corrected only)
    int32_t *status;  // sticky non-finite flag
};

__host__ __device__ constexpr size_t smem_bytes_for(int n, int NT) {
    return sizeof(double) * ((size_t)n + NT / 32 + 1) + sizeof(GmresSmem);
}

// ---------------------------------------------------------------------------
// v = Phi_t(rowbuf) for the CTA's nodes i = tid + k*NT.
// Returns the GMRES Arnoldi count for corrected kinds (-1 on non-finite rhs),
// 0 otherwise.  rowbuf is clobbered for KIND != SL; the caller must
// __syncthreads() before rewriting it.
template <int P, int KIND, int NT, int NPT, bool NUMBA>
__device__ int cta_apply(const mgrit_level_desc &L, int64_t t, const RowCtx &cx,
                         double (&v)[NPT]) {
    constexpr int SL = Stencil<P>::L;
    const int n = L.n_x;
    const int tid = threadIdx.x;
    const int64_t set = L.shared ? 0 : t;
    const double *s = L.s_x + set * (int64_t)n;
    const double *row = cx.rowbuf;

    // ---- semi-Lagrangian gather: left-to-right sum of rounded products
#pragma unroll
    for (int k = 0; k < NPT; ++k) {
        const int i = tid + k * NT;
        double acc = 0.0;
        if (i < n) {
            const Dec d = decompose_s(__ldg(s + i), n);
            double w[P + 1];
            lagrange_weights<P>(d.eps, w);
            int j = d.e - SL;
            if (j < 0) j += n;
#pragma unroll
            for (int c = 0; c <= P; ++c) {
                const double prod = __dmul_rn(row[j], w[c]);
                acc = c == 0 ? prod : __dadd_rn(acc, prod);
                j = (j + 1 == n) ? 0 : j + 1;
            }
        }
        v[k] = acc;
    }
    if constexpr (KIND == MGRIT_KIND_SL) {
        return 0;
    } else {
        constexpr int RAD = (P + 1) / 2;
        const double *sig = L.sig_x + set * (int64_t)n;

        // (I - diag(sig) D) x  on the vector held in rowbuf, at node i
        auto imsd_at = [&](int i, double xi) -> double {
            double acc;
            if constexpr (NUMBA) {
                // _kernels.py:18-31: acc = sum_{k=-rad..rad} st[rad+k] * v[i+k]
                acc = 0.0;
#pragma unroll
                for (int q = -RAD; q <= RAD; ++q) {
                    int j = i + q;
                    j = j < 0 ? j + n : (j >= n ? j - n : j);
                    acc = __dadd_rn(acc, __dmul_rn(dcoef<P>(RAD + q), row[j]));
                }
            } else {
                // coarse_correction.py:50-56: c0 v + sum_k (c_{+k} v_{i+k} + c_{-k} v_{i-k})
                acc = __dmul_rn(dcoef<P>(RAD), xi);
#pragma unroll
                for (int q = 1; q <= RAD; ++q) {
                    int jp = i + q, jm = i - q;
                    jp = jp >= n ? jp - n : jp;
                    jm = jm < 0 ? jm + n : jm;
                    acc = __dadd_rn(acc, __dadd_rn(__dmul_rn(dcoef<P>(RAD + q), row[jp]),
                                                   __dmul_rn(dcoef<P>(RAD - q), row[jm])));
                }
            }
            return __dsub_rn(xi, __dmul_rn(__ldg(sig + i), acc));
        };

        if constexpr (KIND == MGRIT_KIND_FORWARD_EULER) {
            // apply_IpSD (coarse_correction.py:152-154): 2v - (I - diag(sig) D) v
            __syncthreads();
#pragma unroll
            for (int k = 0; k < NPT; ++k) {
                const int i = tid + k * NT;
                if (i < n) cx.rowbuf[i] = v[k];
            }
            __syncthreads();
#pragma unroll
            for (int k = 0; k < NPT; ++k) {
                const int i = tid + k * NT;
                if (i < n) v[k] = __dsub_rn(__dmul_rn(2.0, v[k]), imsd_at(i, v[k]));
            }
            return 0;
        } else {
            // ---- MGS-GMRES, zero start, Givens (coarse_correction.py:173-228,
            //      _kernels.py:34-101) on (I - diag(sig) D) x = v
            const int K = L.gmres_max_iters;
            const double tol = L.gmres_tol;
            GmresSmem &G = *cx.gs;
            double *basis = cx.basis;

            // non-finite rhs -> NaN row + sticky flag (coarse_correction.py:181-182)
            int bad = 0;
#pragma unroll
            for (int k = 0; k < NPT; ++k)
                if (tid + k * NT < n && !isfinite(v[k])) bad = 1;
            if (__syncthreads_or(bad)) {
                if (tid == 0) atomicExch(cx.status, 1);
#pragma unroll
                for (int k = 0; k < NPT; ++k) v[k] = __longlong_as_double(0x7ff8000000000000LL);
                return -1;
            }
            double part = 0.0;
#pragma unroll
            for (int k = 0; k < NPT; ++k) part = __dadd_rn(part, __dmul_rn(v[k], v[k]));
            const double beta = sqrt(block_sum<NT>(part, cx.red));
            if (beta == 0.0) {
#pragma unroll
                for (int k = 0; k < NPT; ++k) v[k] = 0.0;
                return 0;
            }
#pragma unroll
            for (int k = 0; k < NPT; ++k) {
                const int i = tid + k * NT;
                v[k] = __ddiv_rn(v[k], beta);
                if (i < n) basis[i] = v[k];
            }
            if (tid == 0) {
                G.g[0] = beta;
                G.stop = 0;
            }
            int done = 0;
#pragma unroll 1
            for (int kk = 0; kk < K; ++kk) {
                __syncthreads();  // previous users of rowbuf are done
#pragma unroll
                for (int k = 0; k < NPT; ++k) {
                    const int i = tid + k * NT;
                    if (i < n) cx.rowbuf[i] = v[k];  // b_kk
                }
                __syncthreads();
                // w = A b_kk
#pragma unroll
                for (int k = 0; k < NPT; ++k) {
                    const int i = tid + k * NT;
                    v[k] = i < n ? imsd_at(i, row[i]) : 0.0;
                }
                // modified Gram-Schmidt against b_0..b_kk
#pragma unroll 1
                for (int j = 0; j <= kk; ++j) {
                    const double *bj = j == kk ? cx.rowbuf : basis + (int64_t)j * n;
                    double pj = 0.0;
#pragma unroll
                    for (int k = 0; k < NPT; ++k) {
                        const int i = tid + k * NT;
                        if (i < n) pj = __dadd_rn(pj, __dmul_rn(bj[i], v[k]));
                    }
                    const double h = block_sum<NT>(pj, cx.red);
                    if (tid == 0) G.H[j * kMaxKrylov + kk] = h;
#pragma unroll
                    for (int k = 0; k < NPT; ++k) {
                        const int i = tid + k * NT;
                        if (i < n) v[k] = __dsub_rn(v[k], __dmul_rn(h, bj[i]));
                    }
                }
                double pn = 0.0;
#pragma unroll
                for (int k = 0; k < NPT; ++k) pn = __dadd_rn(pn, __dmul_rn(v[k], v[k]));
                const double nrm = sqrt(block_sum<NT>(pn, cx.red));
                const bool brk = nrm <= __dmul_rn(1e-14, beta);
                if (!brk) {
#pragma unroll
                    for (int k = 0; k < NPT; ++k) {
                        const int i = tid + k * NT;
                        v[k] = __ddiv_rn(v[k], nrm);
                        if (i < n) basis[(int64_t)(kk + 1) * n + i] = v[k];
                    }
                }
                if (tid == 0) {
                    double *H = G.H;
                    auto h_ = [&](int a, int b) -> double & { return H[a * kMaxKrylov + b]; };
                    h_(kk + 1, kk) = nrm;
                    for (int j = 0; j < kk; ++j) {
                        const double tmp = __dadd_rn(__dmul_rn(G.cs[j], h_(j, kk)), __dmul_rn(G.sn[j], h_(j + 1, kk)));
                        h_(j + 1, kk) = __dadd_rn(__dmul_rn(-G.sn[j], h_(j, kk)), __dmul_rn(G.cs[j], h_(j + 1, kk)));
                        h_(j, kk) = tmp;
                    }
                    const double den = hypot(h_(kk, kk), h_(kk + 1, kk));
                    G.cs[kk] = __ddiv_rn(h_(kk, kk), den);
                    G.sn[kk] = __ddiv_rn(h_(kk + 1, kk), den);
                    h_(kk, kk) = den;
                    h_(kk + 1, kk) = 0.0;
                    G.g[kk + 1] = __dmul_rn(-G.sn[kk], G.g[kk]);
                    G.g[kk] = __dmul_rn(G.cs[kk], G.g[kk]);
                    G.stop = brk || (tol >= 0.0 && fabs(G.g[kk + 1]) <= __dmul_rn(tol, beta));
                }
                done = kk + 1;
                __syncthreads();
                if (G.stop) break;
            }
            // back substitution (_kernels.py:90-95) on one thread
            if (tid == 0) {
                for (int j = done - 1; j >= 0; --j) {
                    double acc = G.g[j];
                    for (int jj = j + 1; jj < done; ++jj)
                        acc = __dsub_rn(acc, __dmul_rn(G.H[j * kMaxKrylov + jj], G.y[jj]));
                    G.y[j] = __ddiv_rn(acc, G.H[j * kMaxKrylov + j]);
                }
            }
            __syncthreads();
            // x = sum_j b_j y_j (_kernels.py:96-101)
#pragma unroll
            for (int k = 0; k < NPT; ++k) {
                const int i = tid + k * NT;
                double acc = 0.0;
                if (i < n)
                    for (int j = 0; j < done; ++j)
                        acc = __dadd_rn(acc, __dmul_rn(basis[(int64_t)j * n + i], G.y[j]));
                v[k] = acc;
            }
            return done;
        }
    }
}

// store v into rowbuf (after a barrier protecting previous readers)
template <int NT, int NPT>
__device__ __forceinline__ void set_row(double *rowbuf, const double (&v)[NPT], int n) {
    __syncthreads();
#pragma unroll
    for (int k = 0; k < NPT; ++k) {
        const int i = threadIdx.x + k * NT;
        if (i < n) rowbuf[i] = v[k];
    }
    __syncthreads();
}

template <int NT, int NPT>
__device__ __forceinline__ void load_row(double (&v)[NPT], const double *src, int n) {
#pragma unroll
    for (int k = 0; k < NPT; ++k) {
        const int i = threadIdx.x + k * NT;
        v[k] = i < n ? src[i] : 0.0;
    }
}

template <int NT, int NPT>
__device__ __forceinline__ void store_row(double *dst, const double (&v)[NPT], int n) {
#pragma unroll
    for (int k = 0; k < NPT; ++k) {
        const int i = threadIdx.x + k * NT;
        if (i < n) dst[i] = v[k];
    }
}

// v += g (g NULL => + 0.0, keeping the reference's "+ G" rounding of -0.0)
template <int NT, int NPT>
__device__ __forceinline__ void add_forcing(double (&v)[NPT], const double *g, int n) {
#pragma unroll
    for (int k = 0; k < NPT; ++k) {
        const int i = threadIdx.x + k * NT;
        v[k] = __dadd_rn(v[k], (g && i < n) ? g[i] : 0.0);
    }
}

// r = (g + v) - u ; returns this thread's sum of r^2
template <int NT, int NPT>
__device__ __forceinline__ double residual_form(double (&v)[NPT], const double *g, const double *u,
                                                int n) {
    double ss = 0.0;
#pragma unroll
    for (int k = 0; k < NPT; ++k) {
        const int i = threadIdx.x + k * NT;
        if (i < n) {
            const double r = __dsub_rn(__dadd_rn(g ? g[i] : 0.0, v[k]), u[i]);
            v[k] = r;
            ss = __dadd_rn(ss, __dmul_rn(r, r));
        } else {
            v[k] = 0.0;
        }
    }
    return ss;
}

__device__ __forceinline__ RowCtx make_ctx(double *sm, int n, int NT, double *scratch,
                                           int64_t slot, const mgrit_level_desc &L,
                                           int32_t *status) {
    RowCtx c;
    c.rowbuf = sm;
    c.red = sm + n;
    c.gs = reinterpret_cast<GmresSmem *>(sm + n + NT / 32 + 1);
    c.basis = scratch ? scratch + slot * (int64_t)(L.gmres_max_iters + 1) * n : nullptr;
    c.status = status;
    return c;
}

// ---------------------------------------------------------------------------
// apply_rows: one CTA per row (persistent over rows)


template <int P, int KIND, int NT, int NPT>
__global__ void __launch_bounds__(NT) rows_kernel(mgrit_level_desc L, RowsArgs a, double *scratch,
                                                  int32_t *status) {
    extern __shared__ double sm[];
    const int n = L.n_x;
    RowCtx cx = make_ctx(sm, n, NT, scratch, blockIdx.x, L, status);
    for (int64_t b = blockIdx.x; b < a.B; b += gridDim.x) {
        const int64_t t = a.t_idx ? a.t_idx[b] : a.t_first + b * a.t_stride;
        double v[NPT];
        load_row<NT, NPT>(v, a.U_in + b * a.ld_in, n);
        set_row<NT, NPT>(cx.rowbuf, v, n);
        const int cnt = cta_apply<P, KIND, NT, NPT, false>(L, t, cx, v);
        const double *g = a.G ? a.G + b * a.ld_g : nullptr;
        double ss = 0.0;
        if (a.U_sub) {
            ss = residual_form<NT, NPT>(v, g, a.U_sub + b * a.ld_sub, n);
        } else {
            add_forcing<NT, NPT>(v, g, n);
            if (a.row_sumsq)
#pragma unroll
                for (int k = 0; k < NPT; ++k) ss = __dadd_rn(ss, __dmul_rn(v[k], v[k]));
        }
        store_row<NT, NPT>(a.out + b * a.ld_out, v, n);
        if (a.row_sumsq) {
            const double tot = block_sum<NT>(ss, cx.red);
            if (threadIdx.x == 0) a.row_sumsq[b] = tot;
        }
        if (a.gmres_iters && threadIdx.x == 0) a.gmres_iters[b] = cnt;
    }
}

// ---------------------------------------------------------------------------
// fused level phases: one CTA per C-interval (persistent over intervals)

template <int P, int KIND, int NT, int NPT>
__global__ void __launch_bounds__(NT) phase_kernel(mgrit_level_desc L, mgrit_phase_args A,
                                                   double *scratch, int32_t *status) {
    extern __shared__ double sm[];
    const int n = L.n_x;
    const int m = A.m;
    RowCtx cx = make_ctx(sm, n, NT, scratch, blockIdx.x, L, status);
    auto U = [&](int64_t t) { return A.U + (t - A.u_row0) * A.ldu; };
    auto Gr = [&](int64_t t) -> const double * { return A.G ? A.G + (t - A.g_row0) * A.ldg : nullptr; };
    auto Cb = [&](int64_t c) { return A.Cbuf + (c - A.c_row0) * (int64_t)n; };
    auto Ucr = [&](int64_t c) { return A.Uc + (c - A.c_row0) * (int64_t)n; };

    for (int64_t c = A.c_begin + blockIdx.x; c < A.c_begin + A.c_count; c += gridDim.x) {
        const int64_t t0 = c * m;
        const int64_t tC = t0 + m;
        double v[NPT];
        // ---- left state of the interval
        const bool zero_left = A.zero_init && (c == 0 || A.phase == MGRIT_PHASE_FC ||
                                               A.phase == MGRIT_PHASE_FONLY_RES);
        if (zero_left) {
#pragma unroll
            for (int k = 0; k < NPT; ++k) v[k] = 0.0;
            if (c == 0 || A.phase == MGRIT_PHASE_FONLY_RES) store_row<NT, NPT>(U(t0), v, n);
        } else if (A.phase == MGRIT_PHASE_FC || A.phase == MGRIT_PHASE_FONLY_RES || c == 0) {
            load_row<NT, NPT>(v, U(t0), n);
        } else {
            load_row<NT, NPT>(v, Cb(c), n);
        }
        if (A.phase == MGRIT_PHASE_INJ_F) {
            // U[::m] += Uc  (mgrit.py:333)
            double u[NPT];
            load_row<NT, NPT>(u, Ucr(c), n);
#pragma unroll
            for (int k = 0; k < NPT; ++k) v[k] = __dadd_rn(v[k], u[k]);
            store_row<NT, NPT>(U(t0), v, n);
        } else if (A.phase == MGRIT_PHASE_F_RES && c > 0) {
            store_row<NT, NPT>(U(t0), v, n);
        }
        set_row<NT, NPT>(cx.rowbuf, v, n);

        // ---- F-relaxation chain (mgrit.py:276-283) then the interval tail at
        //      k == m; a single call site of the step operator keeps the
        //      kernel body (and its compile time) small.
        const bool last = (c + 1 == A.n_intervals);
        const int kmax = (A.phase == MGRIT_PHASE_INJ_F && !A.partial) ? m - 1 : m;
        if (A.phase == MGRIT_PHASE_INJ_F && !A.partial && last) {
            // U[N] += Uc[N/m] for the final C-point (mgrit.py:333)
            double right[NPT], u[NPT];
            load_row<NT, NPT>(right, Cb(c + 1), n);
            load_row<NT, NPT>(u, Ucr(c + 1), n);
#pragma unroll
            for (int k = 0; k < NPT; ++k) right[k] = __dadd_rn(right[k], u[k]);
            store_row<NT, NPT>(U(tC), right, n);
        }
#pragma unroll 1
        for (int k = 1; k <= kmax; ++k) {
            const int64_t t = t0 + k;
            cta_apply<P, KIND, NT, NPT, false>(L, t - 1, cx, v);
            if (k < m) {
                add_forcing<NT, NPT>(v, Gr(t), n);
                store_row<NT, NPT>(U(t), v, n);
                set_row<NT, NPT>(cx.rowbuf, v, n);
                continue;
            }
            // ---- interval tail at the right C-point tC = t
            if (A.phase == MGRIT_PHASE_FC) {
                // C-relaxation (mgrit.py:286-290) into the C-point buffer
                add_forcing<NT, NPT>(v, Gr(tC), n);
                store_row<NT, NPT>(Cb(c + 1), v, n);
                break;
            }
            // subtrahend of the C-point residual: the current U[tC]
            double right[NPT];
            if (A.phase == MGRIT_PHASE_INJ_F) {
                double u[NPT];
                load_row<NT, NPT>(right, Cb(c + 1), n);
                load_row<NT, NPT>(u, Ucr(c + 1), n);
#pragma unroll
                for (int q = 0; q < NPT; ++q) right[q] = __dadd_rn(right[q], u[q]);
                if (last) store_row<NT, NPT>(U(tC), right, n);
            } else if (A.phase == MGRIT_PHASE_F_RES) {
                load_row<NT, NPT>(right, Cb(c + 1), n);
                store_row<NT, NPT>(U(tC), right, n);
            } else {  // FONLY_RES
                if (A.zero_init) {
#pragma unroll
                    for (int q = 0; q < NPT; ++q) right[q] = 0.0;
                    store_row<NT, NPT>(U(tC), right, n);
                } else {
                    load_row<NT, NPT>(right, U(tC), n);
                }
                store_row<NT, NPT>(Cb(c + 1), right, n);
            }
            // r = (G + Phi U[tC-1]) - U[tC]; F-point residuals are exactly 0
            // after F-relaxation ((G + S) - (S + G) == 0 bitwise), so the
            // restriction Gc = R[::m] and the norm only need C-points.
            double ss = 0.0;
            const double *g = Gr(tC);
#pragma unroll
            for (int q = 0; q < NPT; ++q) {
                const int i = threadIdx.x + q * NT;
                if (i < n) {
                    const double r = __dsub_rn(__dadd_rn(g ? g[i] : 0.0, v[q]), right[q]);
                    v[q] = r;
                    ss = __dadd_rn(ss, __dmul_rn(r, r));
                }
            }
            if (A.Gc && A.phase != MGRIT_PHASE_INJ_F)
                store_row<NT, NPT>(A.Gc + (c + 1 - A.c_row0) * (int64_t)n, v, n);
            if (A.partial) {
                const double tot = block_sum<NT>(ss, cx.red);
                if (threadIdx.x == 0) A.partial[c - A.partial0] = tot;
            }
        }
    }
}

// ---------------------------------------------------------------------------
// sequential sweep: one CTA steps the whole level

template <int P, int KIND, int NT, int NPT, bool NUMBA>
__global__ void __launch_bounds__(NT) sweep_kernel(mgrit_level_desc L, double *U, int64_t ldu,
                                                   const double *G, int64_t ldg, int zero_init,
                                                   int32_t *gmres_iters, double *scratch,
                                                   int32_t *status) {
    extern __shared__ double sm[];
    const int n = L.n_x;
    RowCtx cx = make_ctx(sm, n, NT, scratch, 0, L, status);
    double v[NPT];
    if (zero_init) {
#pragma unroll
        for (int k = 0; k < NPT; ++k) v[k] = 0.0;
        store_row<NT, NPT>(U, v, n);
    } else {
        load_row<NT, NPT>(v, U, n);
    }
    set_row<NT, NPT>(cx.rowbuf, v, n);
    for (int64_t t = 0; t < L.n_steps; ++t) {
        const int cnt = cta_apply<P, KIND, NT, NPT, NUMBA>(L, t, cx, v);
        add_forcing<NT, NPT>(v, G ? G + (t + 1) * ldg : nullptr, n);
        store_row<NT, NPT>(U + (t + 1) * ldu, v, n);
        if (gmres_iters && threadIdx.x == 0) gmres_iters[t] = cnt;
        set_row<NT, NPT>(cx.rowbuf, v, n);
    }
}

// ---------------------------------------------------------------------------
// launch configuration: a CTA owns a whole row, NPT <= 16 nodes per thread

struct Cfg1D {
    int nt, npt;
};

static Cfg1D cfg_for(int n) {
    if (n <= 2048) return {128, 16};
    if (n <= 4096) return {256, 16};
    if (n <= 8192) return {512, 16};
    return {512, 32};
}

static int resident_ctas(const void *fn, int nt, size_t smem) {
    int dev = 0, sms = 148, per = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fn, nt, smem) != cudaSuccess || per < 1)
        per = 1;
    return sms * per;
}

template <typename F>
static int prep(F fn, size_t smem) {
    static_assert(sizeof(F) > 0, "");
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute((const void *)fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem);
        if (e != cudaSuccess) {
            set_error("cudaFuncSetAttribute", e);
            return MGRIT_ECUDA;
        }
    }
    return MGRIT_OK;
}

template <int P_, int KIND_, int NT_, int NPT_>
struct Tag {
    static constexpr int P = P_, KIND = KIND_, NT = NT_, NPT = NPT_;
};

template <int P, int KIND, typename F>
static int dispatch_cfg(Cfg1D c, F &&f) {
    if (c.nt <= 128) return f(Tag<P, KIND, 128, 16>{});
    if (c.nt <= 256) return f(Tag<P, KIND, 256, 16>{});
    if (c.npt <= 16) return f(Tag<P, KIND, 512, 16>{});
    return f(Tag<P, KIND, 512, 32>{});
}

inline int validate(const mgrit_level_desc *L) {
    if (!L || L->dim != 1 || L->n_x < 1 || L->n_x > 16384 || !L->s_x) return MGRIT_EINVAL;
    if (L->p != 1 && L->p != 3 && L->p != 5) return MGRIT_EINVAL;
    if (L->kind < 0 || L->kind > 2) return MGRIT_EINVAL;
    if (L->kind != MGRIT_KIND_SL && !L->sig_x) return MGRIT_EINVAL;
    if (L->kind == MGRIT_KIND_CORRECTED && (L->gmres_max_iters < 1 || L->gmres_max_iters > kMaxKrylov))
        return MGRIT_EINVAL;
    return MGRIT_OK;
}

inline int64_t scratch_per_cta(const mgrit_level_desc *L) {
    return L->kind == MGRIT_KIND_CORRECTED ? (int64_t)(L->gmres_max_iters + 1) * L->n_x * 8 : 0;
}

inline int cap_grid(int64_t want, int resident, const mgrit_level_desc *L, int64_t scratch_bytes) {
    int64_t g = want < resident ? want : resident;
    const int64_t per = scratch_per_cta(L);
    if (per > 0) {
        const int64_t fit = scratch_bytes / per;
        if (fit < g) g = fit;
    }
    return (int)g;
}


// Host launchers for one (P, KIND); explicitly instantiated one pair per
// translation unit (step1d_p*_k*.cu) so the heavy kernel bodies compile in
// parallel.
template <int P, int KIND>
struct Launch1D {
    static int64_t capacity(const mgrit_level_desc *L);
    static int rows(const mgrit_level_desc *L, const RowsArgs &a, void *scratch,
                    int64_t scratch_bytes, int32_t *status, cudaStream_t st);
    static int phase(const mgrit_level_desc *L, const mgrit_phase_args *A, void *scratch,
                     int64_t scratch_bytes, int32_t *status, cudaStream_t st);
    static int sweep(const mgrit_level_desc *L, double *U, int64_t ldu, const double *G,
                     int64_t ldg, int zero_init, int32_t *gmres_iters, void *scratch,
                     int64_t scratch_bytes, int32_t *status, cudaStream_t st);
};

#ifdef MGRIT_LAUNCH1D_IMPL
template <int P, int KIND>
int64_t Launch1D<P, KIND>::capacity(const mgrit_level_desc *L) {
    const Cfg1D c = cfg_for(L->n_x);
    const size_t smem = smem_bytes_for(L->n_x, c.nt);
    return dispatch_cfg<P, KIND>(c, [&](auto T) {
        using C = decltype(T);
        return resident_ctas((const void *)rows_kernel<C::P, C::KIND, C::NT, C::NPT>, C::NT, smem);
    });
}

template <int P, int KIND>
int Launch1D<P, KIND>::rows(const mgrit_level_desc *L, const RowsArgs &a, void *scratch,
                  int64_t scratch_bytes, int32_t *status, cudaStream_t st) {
    int rc = validate(L);
    if (rc) return rc;
    if (a.B <= 0) return MGRIT_OK;
    const Cfg1D c = cfg_for(L->n_x);
    const size_t smem = smem_bytes_for(L->n_x, c.nt);
    rc = dispatch_cfg<P, KIND>(c, [&](auto T) {
        using C = decltype(T);
        auto fn = rows_kernel<C::P, C::KIND, C::NT, C::NPT>;
        int r = prep(fn, smem);
        if (r) return r;
        const int grid = cap_grid(a.B, resident_ctas((const void *)fn, C::NT, smem), L, scratch_bytes);
        if (grid < 1) return (int)MGRIT_EINVAL;
        fn<<<grid, C::NT, smem, st>>>(*L, a, (double *)scratch, status);
        return (int)MGRIT_OK;
    });
    if (rc) return rc;
    return check_launch("apply_rows");
}

template <int P, int KIND>
int Launch1D<P, KIND>::phase(const mgrit_level_desc *L, const mgrit_phase_args *A, void *scratch,
                   int64_t scratch_bytes, int32_t *status, cudaStream_t st) {
    int rc = validate(L);
    if (rc) return rc;
    if (!A || A->m < 1 || !A->U || A->c_count < 0 || A->n_intervals < 1) return MGRIT_EINVAL;
    if ((int64_t)A->n_intervals * A->m != L->n_steps) return MGRIT_EINVAL;
    if (A->phase < 0 || A->phase > 3) return MGRIT_EINVAL;
    if (!A->Cbuf) return MGRIT_EINVAL;
    if (A->phase == MGRIT_PHASE_INJ_F && !A->Uc) return MGRIT_EINVAL;
    if (A->c_count == 0) return MGRIT_OK;
    const Cfg1D c = cfg_for(L->n_x);
    const size_t smem = smem_bytes_for(L->n_x, c.nt);
    rc = dispatch_cfg<P, KIND>(c, [&](auto T) {
        using C = decltype(T);
        auto fn = phase_kernel<C::P, C::KIND, C::NT, C::NPT>;
        int r = prep(fn, smem);
        if (r) return r;
        const int grid = cap_grid(A->c_count, resident_ctas((const void *)fn, C::NT, smem), L, scratch_bytes);
        if (grid < 1) return (int)MGRIT_EINVAL;
        fn<<<grid, C::NT, smem, st>>>(*L, *A, (double *)scratch, status);
        return (int)MGRIT_OK;
    });
    if (rc) return rc;
    return check_launch("level_phase");
}

template <int P, int KIND>
int Launch1D<P, KIND>::sweep(const mgrit_level_desc *L, double *U, int64_t ldu, const double *G, int64_t ldg,
             int zero_init, int32_t *gmres_iters, void *scratch, int64_t scratch_bytes,
             int32_t *status, cudaStream_t st) {
    int rc = validate(L);
    if (rc) return rc;
    if (!U) return MGRIT_EINVAL;
    if (scratch_per_cta(L) > scratch_bytes) return MGRIT_EINVAL;
    const Cfg1D c = cfg_for(L->n_x);
    const size_t smem = smem_bytes_for(L->n_x, c.nt);
    const bool numba = L->stencil_numba && L->kind == MGRIT_KIND_CORRECTED;
    rc = dispatch_cfg<P, KIND>(c, [&](auto T) {
        using C = decltype(T);
        int r;
        if constexpr (C::KIND == MGRIT_KIND_CORRECTED) {
            if (numba) {
                auto fn = sweep_kernel<C::P, C::KIND, C::NT, C::NPT, true>;
                if ((r = prep(fn, smem))) return r;
                fn<<<1, C::NT, smem, st>>>(*L, U, ldu, G, ldg, zero_init, gmres_iters, (double *)scratch, status);
                return (int)MGRIT_OK;
            }
        }
        auto fn = sweep_kernel<C::P, C::KIND, C::NT, C::NPT, false>;
        if ((r = prep(fn, smem))) return r;
        fn<<<1, C::NT, smem, st>>>(*L, U, ldu, G, ldg, zero_init, gmres_iters, (double *)scratch, status);
        return (int)MGRIT_OK;
    });
    if (rc) return rc;
    return check_launch("sequential_sweep");
}

#endif  // MGRIT_LAUNCH1D_IMPL

}  // namespace mgrit
