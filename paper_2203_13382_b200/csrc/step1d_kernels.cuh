// step1d_kernels.cuh — the 1D hot path: batched SL / corrected / forward-Euler step
// operators and the fused MGRIT level phases.
//
// Design (B200): a 1D state row (n <= 16384 fp64 = 128 KB) fits in one SM's
// shared memory, so a CTA owns a whole row.  The fused phase kernels give one
// CTA per C-interval and walk its m-1 dependent F-steps with the state kept
// in shared memory: per step only the departure record (8 B/node) is read
// (prefetched into registers one step ahead) and the new state (8 B/node)
// written to HBM; the previous state never round-trips through HBM.
//
// The corrected operator's MGS-GMRES runs inside the CTA: the first Krylov
// vectors live in shared memory next to the state row (the rest spill to a
// per-CTA L2-resident slab), sigma stays in registers, dot products use four
// independent accumulator chains, block reductions are double-buffered (two
// barriers each), and the 1/beta, 1/h_{k+1,k} scalings use one correctly
// rounded reciprocal plus an exact FMA correction per element (Markstein),
// which is bit-identical to the division.  Grids are persistent
// (<= resident-CTA capacity), looping over rows / intervals.
#include "internal.cuh"

namespace mgrit {

constexpr int kMaxKrylov = 16;

#ifdef MGRIT_PROBE
// clock64 timestamps of CTA 0 / thread 0 (tools/probe_gmres.cu only)
__device__ long long g_probe[512];
#define MGRIT_PROBE_AT(id) \
    do { if (threadIdx.x == 0 && blockIdx.x == 0 && (id) < 512) g_probe[(id)] = clock64(); } while (0)
#else
#define MGRIT_PROBE_AT(id) do {} while (0)
#endif
// periodic halo kept on both sides of the shared-memory row so stencil taps
// (<= 3 cells: p = 5 interpolation, D_6) need no wrap-around arithmetic
constexpr int kHalo = 4;

// row[i] = x plus its periodic halo image (row[-kHalo..-1], row[n..n+kHalo-1])
__device__ __forceinline__ void put_row(double *row, int i, double x, int n) {
    row[i] = x;
    if (i < kHalo) row[n + i] = x;
    if (i >= n - kHalo) row[i - n] = x;
}

// per-CTA GMRES control block + reduction buffers in shared memory
struct GmresSmem {
    double H[(kMaxKrylov + 1) * kMaxKrylov];
    double cs[kMaxKrylov], sn[kMaxKrylov], g[kMaxKrylov + 1], y[kMaxKrylov];
    double red[2][33];
    int stop;
};

struct RowCtx {
    double *rowbuf;   // smem, n doubles: state row / Krylov vector for the stencil
    GmresSmem *gs;    // smem
    double *bsm;      // smem Krylov slots [nbs][n]
    double *bgl;      // global Krylov slots [(K+1-nbs)][n] (corrected only)
    int nbs;
    int sel;          // double-buffer parity of the block reductions
    int32_t *status;  // sticky non-finite flag
    double *hist;     // nullable: GMRES residual history [K+1] of the current row
    __device__ __forceinline__ double *bvec(int j, int n) const {
        return j < nbs ? bsm + (int64_t)j * n : bgl + (int64_t)(j - nbs) * n;
    }
};

// Fixed-order pairwise sum of N doubles in shared memory (broadcast reads).
template <int N>
__device__ __forceinline__ double tree_sum(const double *r) {
    if constexpr (N == 1) {
        return r[0];
    } else {
        return __dadd_rn(tree_sum<N / 2>(r), tree_sum<N - N / 2>(r + N / 2));
    }
}

// Block-wide fixed-order sum, one barrier: warp butterflies, then every
// warp reduces the NT/32 warp partials with the same butterfly.  The
// scratch is double-buffered by call parity: call c+2 reuses call c's slots
// only after every thread has passed call c+1's barrier.
template <int NT>
__device__ __forceinline__ double block_sum2(double v, RowCtx &cx) {
    constexpr int NW = NT / 32;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double *red = cx.gs->red[cx.sel];
    cx.sel ^= 1;
    v = warp_sum(v);
    if (lane == 0) red[warp] = v;
    __syncthreads();
    if constexpr (NW <= 8) {
        return tree_sum<NW>(red);  // few partials: broadcast loads + pairwise tree
    } else {
        return warp_sum(lane < NW ? red[lane] : 0.0);
    }
}


template <int NT, int NPT, bool F>
__device__ __forceinline__ void load_records(const mgrit_level_desc &L, int64_t t, double (&sv)[NPT]) {
    const int n = L.n_x;
    const double *s = L.s_x + (L.shared ? 0 : t) * (int64_t)n;
#pragma unroll
    for (int k = 0; k < NPT; ++k) {
        const int i = threadIdx.x + k * NT;
        sv[k] = (F || i < n) ? __ldg(s + i) : 0.0;
    }
}

// ---------------------------------------------------------------------------
// v = Phi_t(rowbuf) for the CTA's nodes i = tid + k*NT, records preloaded in sv.
// Returns the GMRES Arnoldi count for corrected kinds (-1 on non-finite rhs),
// 0 otherwise.  rowbuf is clobbered for KIND != SL; the caller must
// __syncthreads() before rewriting it.
template <int P, int KIND, int NT, int NPT, bool F, bool NUMBA, bool LOWREG = false>
__device__ int cta_apply(const mgrit_level_desc &L, int64_t t, RowCtx &cx, double (&v)[NPT],
                         const double (&sv)[NPT]) {
    constexpr int SL = Stencil<P>::L;
    const int n = L.n_x;
    const int tid = threadIdx.x;
    const double *row = cx.rowbuf;

    // ---- semi-Lagrangian gather: left-to-right sum of rounded products
    MGRIT_PROBE_AT(0);
#pragma unroll
    for (int k = 0; k < NPT; ++k) {
        const int i = tid + k * NT;
        double acc = 0.0;
        if (F || i < n) {
            const Dec d = decompose_s(sv[k], n);
            double w[P + 1];
            lagrange_weights<P>(d.eps, w);
            const double *src = row + (d.e - SL);  // halo covers e-SL >= -3, e+R <= n+1
#pragma unroll
            for (int c = 0; c <= P; ++c) {
                const double prod = __dmul_rn(src[c], w[c]);
                acc = c == 0 ? prod : __dadd_rn(acc, prod);
            }
        }
        v[k] = acc;
    }
    if constexpr (KIND == MGRIT_KIND_SL) {
        return 0;
    } else {
        constexpr int RAD = (P + 1) / 2;
        // sigma in registers unless the kernel runs two CTAs per SM (LOWREG)
        constexpr bool SIGREG = !LOWREG && (NPT <= 8 || NT <= 256);
        const int64_t set = L.shared ? 0 : t;
        const double *sig = L.sig_x + set * (int64_t)n;
        double sg[SIGREG ? NPT : 1];
        if constexpr (SIGREG) {
#pragma unroll
            for (int k = 0; k < NPT; ++k) {
                const int i = tid + k * NT;
                sg[k] = (F || i < n) ? __ldg(sig + i) : 0.0;
            }
        }
        // (I - diag(sig) D) x at node i (k-th node of this thread) on rowbuf
        auto imsd_at = [&](int k, int i, double xi) -> double {
            double acc;
            if constexpr (NUMBA) {
                // _kernels.py:18-31: acc = sum_{k=-rad..rad} st[rad+k] * v[i+k]
                acc = 0.0;
#pragma unroll
                for (int q = -RAD; q <= RAD; ++q)
                    acc = __dadd_rn(acc, cmul<P>(RAD + q, row[i + q]));
            } else {
                // coarse_correction.py:50-56: c0 v + sum_k (c_{+k} v_{i+k} + c_{-k} v_{i-k})
                acc = cmul<P>(RAD, xi);
#pragma unroll
                for (int q = 1; q <= RAD; ++q)
                    acc = __dadd_rn(acc, __dadd_rn(cmul<P>(RAD + q, row[i + q]), cmul<P>(RAD - q, row[i - q])));
            }
            double s_i;
            if constexpr (SIGREG) s_i = sg[k];
            else s_i = __ldg(sig + i);
            return __dsub_rn(xi, __dmul_rn(s_i, acc));
        };

        if constexpr (KIND == MGRIT_KIND_FORWARD_EULER) {
            // apply_IpSD (coarse_correction.py:152-154): 2v - (I - diag(sig) D) v
            __syncthreads();
#pragma unroll
            for (int k = 0; k < NPT; ++k) {
                const int i = tid + k * NT;
                if (F || i < n) put_row(cx.rowbuf, i, v[k], n);
            }
            __syncthreads();
#pragma unroll
            for (int k = 0; k < NPT; ++k) {
                const int i = tid + k * NT;
                if (F || i < n) v[k] = __dsub_rn(__dmul_rn(2.0, v[k]), imsd_at(k, i, v[k]));
            }
            return 0;
        } else {
            // ---- MGS-GMRES, zero start, Givens (coarse_correction.py:173-228,
            //      _kernels.py:34-101) on (I - diag(sig) D) x = v.
            // The operator application is the reference's exact arithmetic;
            // inner products / axpys use FMA (their reference counterparts are
            // BLAS calls whose rounding is not reproducible anyway).
            const int K = L.gmres_max_iters;
            const double tol = L.gmres_tol;
            GmresSmem &G = *cx.gs;

            // non-finite rhs -> NaN row + sticky flag (coarse_correction.py:181-182)
            int bad = 0;
#pragma unroll
            for (int k = 0; k < NPT; ++k)
                if ((F || tid + k * NT < n) && !isfinite(v[k])) bad = 1;
            if (__syncthreads_or(bad)) {
                if (tid == 0) atomicExch(cx.status, 1);
#pragma unroll
                for (int k = 0; k < NPT; ++k) v[k] = __longlong_as_double(0x7ff8000000000000LL);
                return -1;
            }
            auto sumsq4 = [&]() -> double {
                double a[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
                for (int k = 0; k < NPT; ++k) a[k & 3] = fma(v[k], v[k], a[k & 3]);
                return __dadd_rn(__dadd_rn(a[0], a[1]), __dadd_rn(a[2], a[3]));
            };
            MGRIT_PROBE_AT(1);
            const double beta = sqrt(block_sum2<NT>(sumsq4(), cx));
            MGRIT_PROBE_AT(2);
            if (cx.hist && tid == 0) cx.hist[0] = beta;
            if (beta == 0.0) {
#pragma unroll
                for (int k = 0; k < NPT; ++k) v[k] = 0.0;
                return 0;
            }
            {
                const double yb = 1.0 / beta;
                double *b0 = cx.bvec(0, n);
#pragma unroll
                for (int k = 0; k < NPT; ++k) {
                    const int i = tid + k * NT;
                    v[k] = div_rcp(v[k], beta, yb);
                    if (F || i < n) b0[i] = v[k];
                }
            }
            double g_k = beta;  // running g[kk] of the least-squares rhs (every thread)
            int done = 0;
#pragma unroll 1
            for (int kk = 0; kk < K; ++kk) {
                MGRIT_PROBE_AT(10 + 8 * kk);
                __syncthreads();  // previous users of rowbuf are done
#pragma unroll
                for (int k = 0; k < NPT; ++k) {
                    const int i = tid + k * NT;
                    if (F || i < n) put_row(cx.rowbuf, i, v[k], n);  // b_kk
                }
                __syncthreads();
                // w = A b_kk
#pragma unroll
                for (int k = 0; k < NPT; ++k) {
                    const int i = tid + k * NT;
                    v[k] = (F || i < n) ? imsd_at(k, i, v[k]) : 0.0;
                }
                MGRIT_PROBE_AT(11 + 8 * kk);
                // modified Gram-Schmidt against b_0..b_kk (b_kk read from rowbuf);
                // b_{j+1} is fetched into registers while b_j's reduction runs.
                // Thread 0 applies the previous Givens rotations to column kk as
                // its entries arrive (rotation j needs h_j and h_{j+1} only), in
                // the reference's order.
                double hrun = 0.0;  // column kk entry j after rotations < j (every thread)
                double bc[NPT];
                {
                    const double *b0p = kk == 0 ? cx.rowbuf : cx.bvec(0, n);
#pragma unroll
                    for (int k = 0; k < NPT; ++k) {
                        const int i = tid + k * NT;
                        bc[k] = (F || i < n) ? b0p[i] : 0.0;
                    }
                }
                // one MGS step on (cur = b_j in registers); nxt receives b_{j+1}
                // (loads issued first so they overlap the FMAs and the reduction)
                auto mgs_step = [&](int j, double (&cur)[NPT], double (&nxt)[NPT]) {
                    if constexpr (LOWREG) {
                        // no register prefetch of b_{j+1} (register budget of two
                        // CTAs per SM): load b_j here; the co-resident CTA hides
                        // the shared-memory latency
                        if (j > 0) {
                            const double *bp = j == kk ? cx.rowbuf : cx.bvec(j, n);
#pragma unroll
                            for (int k = 0; k < NPT; ++k) {
                                const int i = tid + k * NT;
                                cur[k] = (F || i < n) ? bp[i] : 0.0;
                            }
                        }
                    } else if (j < kk) {
                        const double *bp = j + 1 == kk ? cx.rowbuf : cx.bvec(j + 1, n);
#pragma unroll
                        for (int k = 0; k < NPT; ++k) {
                            const int i = tid + k * NT;
                            nxt[k] = (F || i < n) ? bp[i] : 0.0;
                        }
                    }
                    double a4[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
                    for (int k = 0; k < NPT; ++k) a4[k & 3] = fma(cur[k], v[k], a4[k & 3]);
                    const double part = __dadd_rn(__dadd_rn(a4[0], a4[1]), __dadd_rn(a4[2], a4[3]));
                    double c = 0.0, sn = 0.0;
                    if (j > 0) {
                        c = G.cs[j - 1];
                        sn = G.sn[j - 1];
                    }
                    if (kk == 5) MGRIT_PROBE_AT(301 + 4 * j);
                    const double h = block_sum2<NT>(part, cx);
                    if (kk == 5) MGRIT_PROBE_AT(302 + 4 * j);
                    // every thread applies the rotations (identical inputs ->
                    // identical values), so the stop test needs no barrier
                    if (j == 0) {
                        hrun = h;
                    } else {
                        // rotation j-1 on rows (j-1, j) of column kk
                        const double tmp = __dadd_rn(__dmul_rn(c, hrun), __dmul_rn(sn, h));
                        hrun = __dadd_rn(__dmul_rn(-sn, hrun), __dmul_rn(c, h));
                        if (tid == 0) G.H[(j - 1) * kMaxKrylov + kk] = tmp;
                    }
#pragma unroll
                    for (int k = 0; k < NPT; ++k) v[k] = fma(-h, cur[k], v[k]);
                    if (kk == 5) MGRIT_PROBE_AT(303 + 4 * j);
                };
                if constexpr (LOWREG) {
#pragma unroll 1
                    for (int j = 0; j <= kk; ++j) mgs_step(j, bc, bc);
                } else {
                    double bo[NPT];
#pragma unroll 1
                    for (int j = 0; j <= kk; j += 2) {
                        mgs_step(j, bc, bo);
                        if (j + 1 <= kk) mgs_step(j + 1, bo, bc);
                    }
                }
                MGRIT_PROBE_AT(12 + 8 * kk);
                const double nrm = sqrt(block_sum2<NT>(sumsq4(), cx));
                MGRIT_PROBE_AT(13 + 8 * kk);
                const bool brk = nrm <= __dmul_rn(1e-14, beta);
                // new rotation from (H[kk][kk], h_{kk+1,kk} = nrm), evaluated
                // by every thread; the divisions are reciprocal + Markstein
                // correction (correctly rounded, = hess / denom).  b_{kk+1} =
                // w / h_{kk+1,kk} below is written even on breakdown (the slot
                // is then never read), so no branch separates the two chains.
                bool stop;
                {
                    const double den = hypot(hrun, nrm);
                    const double rden = __drcp_rn(den);
                    const double c = div_rcp(hrun, den, rden), sn = div_rcp(nrm, den, rden);
                    const double gn = __dmul_rn(-sn, g_k);
                    if (tid == 0) {
                        G.cs[kk] = c;
                        G.sn[kk] = sn;
                        G.H[kk * kMaxKrylov + kk] = den;
                        G.g[kk] = __dmul_rn(c, g_k);
                        G.g[kk + 1] = gn;
                        if (cx.hist) cx.hist[kk + 1] = fabs(gn);
                    }
                    g_k = gn;
                    stop = brk || (tol >= 0.0 && fabs(gn) <= __dmul_rn(tol, beta));
                }
                MGRIT_PROBE_AT(14 + 8 * kk);
                {
                    const double yn = __drcp_rn(nrm);
                    double *bnv = cx.bvec(kk + 1, n);
#pragma unroll
                    for (int k = 0; k < NPT; ++k) {
                        const int i = tid + k * NT;
                        v[k] = div_rcp(v[k], nrm, yn);
                        if (F || i < n) bnv[i] = v[k];
                    }
                }
                MGRIT_PROBE_AT(15 + 8 * kk);
                done = kk + 1;
                MGRIT_PROBE_AT(16 + 8 * kk);
                if (stop) break;
            }
            __syncthreads();  // G.H / G.g from thread 0
            // back substitution on warp 0 (column-oriented, as LAPACK trsv):
            // lane i keeps acc_i = g_i - sum_{j>i} H[i][j] y_j
            if (tid < 32) {
                const int lane = tid;
                double acc = lane < done ? G.g[lane] : 0.0;
                for (int j = done - 1; j >= 0; --j) {
                    double yj = 0.0;
                    if (lane == j) yj = __ddiv_rn(acc, G.H[j * kMaxKrylov + j]);
                    yj = __shfl_sync(0xffffffffu, yj, j);
                    if (lane == j) G.y[j] = yj;
                    if (lane < j) acc = __dsub_rn(acc, __dmul_rn(G.H[lane * kMaxKrylov + j], yj));
                }
            }
            __syncthreads();
            MGRIT_PROBE_AT(200);
            // x = sum_j b_j y_j (_kernels.py:96-101), j ascending per node
#pragma unroll
            for (int k = 0; k < NPT; ++k) v[k] = 0.0;
#pragma unroll 1
            for (int j = 0; j < done; ++j) {
                const double yj = G.y[j];
                const double *bj = cx.bvec(j, n);
#pragma unroll
                for (int k = 0; k < NPT; ++k) {
                    const int i = tid + k * NT;
                    if (F || i < n) v[k] = fma(bj[i], yj, v[k]);
                }
            }
            MGRIT_PROBE_AT(201);
            return done;
        }
    }
}

// store v into rowbuf (after a barrier protecting previous readers)
template <int NT, int NPT, bool F>
__device__ __forceinline__ void set_row(double *rowbuf, const double (&v)[NPT], int n) {
    __syncthreads();
#pragma unroll
    for (int k = 0; k < NPT; ++k) {
        const int i = threadIdx.x + k * NT;
        if (F || i < n) put_row(rowbuf, i, v[k], n);
    }
    __syncthreads();
}

template <int NT, int NPT, bool F>
__device__ __forceinline__ void load_row(double (&v)[NPT], const double *src, int n) {
#pragma unroll
    for (int k = 0; k < NPT; ++k) {
        const int i = threadIdx.x + k * NT;
        v[k] = (F || i < n) ? src[i] : 0.0;
    }
}

template <int NT, int NPT, bool F>
__device__ __forceinline__ void store_row(double *dst, const double (&v)[NPT], int n) {
#pragma unroll
    for (int k = 0; k < NPT; ++k) {
        const int i = threadIdx.x + k * NT;
        if (F || i < n) dst[i] = v[k];
    }
}

// v += g (g NULL => + 0.0, keeping the reference's "+ G" rounding of -0.0)
template <int NT, int NPT, bool F>
__device__ __forceinline__ void add_forcing(double (&v)[NPT], const double *g, int n) {
#pragma unroll
    for (int k = 0; k < NPT; ++k) {
        const int i = threadIdx.x + k * NT;
        v[k] = __dadd_rn(v[k], (g && (F || i < n)) ? g[i] : 0.0);
    }
}

// r = (g + v) - u ; returns this thread's sum of r^2
template <int NT, int NPT, bool F>
__device__ __forceinline__ double residual_form(double (&v)[NPT], const double *g, const double *u,
                                                int n) {
    double ss = 0.0;
#pragma unroll
    for (int k = 0; k < NPT; ++k) {
        const int i = threadIdx.x + k * NT;
        if (F || i < n) {
            const double r = __dsub_rn(__dadd_rn(g ? g[i] : 0.0, v[k]), u[i]);
            v[k] = r;
            ss = __dadd_rn(ss, __dmul_rn(r, r));
        } else {
            v[k] = 0.0;
        }
    }
    return ss;
}

// dynamic shared memory: [halo | rowbuf n | halo][GmresSmem][nbs slots of n][2*kHalo]
__host__ __device__ inline size_t smem_bytes_for(int n, int nbs) {
    // the trailing 2*kHalo doubles give the SL path's second row buffer its halo
    return sizeof(double) * ((size_t)n + 2 * kHalo) + sizeof(GmresSmem) +
           sizeof(double) * ((size_t)n * nbs + 2 * kHalo);
}

__device__ __forceinline__ RowCtx make_ctx(double *sm, int n, int nbs, double *scratch, int64_t slot,
                                           const mgrit_level_desc &L, int32_t *status) {
    RowCtx c;
    c.rowbuf = sm + kHalo;
    c.gs = reinterpret_cast<GmresSmem *>(sm + n + 2 * kHalo);
    c.bsm = reinterpret_cast<double *>(c.gs + 1);
    c.nbs = nbs;
    const int spill = L.gmres_max_iters + 1 - nbs;
    c.bgl = (scratch && spill > 0) ? scratch + slot * (int64_t)spill * n : nullptr;
    c.sel = 0;
    c.status = status;
    c.hist = nullptr;
    return c;
}

// ---------------------------------------------------------------------------
// apply_rows: one CTA per row (persistent over rows)

template <int P, int KIND, int NT, int NPT, bool F>
__global__ void __launch_bounds__(NT, 1) rows_kernel(mgrit_level_desc L, RowsArgs a, int nbs, double *scratch,
                                                  int32_t *status) {
    extern __shared__ double sm[];
    const int n = L.n_x;
    RowCtx cx = make_ctx(sm, n, nbs, scratch, blockIdx.x, L, status);
    for (int64_t b = blockIdx.x; b < a.B; b += gridDim.x) {
        const int64_t t = a.t_idx ? a.t_idx[b] : a.t_first + b * a.t_stride;
        double v[NPT], sv[NPT];
        load_records<NT, NPT, F>(L, t, sv);
        load_row<NT, NPT, F>(v, a.U_in + b * a.ld_in, n);
        set_row<NT, NPT, F>(cx.rowbuf, v, n);
        cx.hist = a.gmres_hist ? a.gmres_hist + b * (int64_t)(L.gmres_max_iters + 1) : nullptr;
        const int cnt = cta_apply<P, KIND, NT, NPT, F, false>(L, t, cx, v, sv);
        const double *g = a.G ? a.G + b * a.ld_g : nullptr;
        double ss = 0.0;
        if (a.U_sub) {
            ss = residual_form<NT, NPT, F>(v, g, a.U_sub + b * a.ld_sub, n);
        } else {
            add_forcing<NT, NPT, F>(v, g, n);
            if (a.row_sumsq)
#pragma unroll
                for (int k = 0; k < NPT; ++k) ss = __dadd_rn(ss, __dmul_rn(v[k], v[k]));
        }
        if (a.out) store_row<NT, NPT, F>(a.out + b * a.ld_out, v, n);
        if (a.row_sumsq) {
            const double tot = block_sum2<NT>(ss, cx);
            if (threadIdx.x == 0) a.row_sumsq[b] = tot;
        }
        if (a.gmres_iters && threadIdx.x == 0) a.gmres_iters[b] = cnt;
    }
}

// ---------------------------------------------------------------------------
// fused level phases: one CTA per C-interval (persistent over intervals)

template <int P, int KIND, int NT, int NPT, bool F, int MINB = 1>
__global__ void __launch_bounds__(NT, MINB) phase_kernel(mgrit_level_desc L, mgrit_phase_args A, int nbs,
                                                      double *scratch, int32_t *status) {
    extern __shared__ double sm[];
    // The next step's departure records are prefetched into registers while
    // the current step computes (plain SL and small NPT; register prefetch
    // measured faster than cp.async staging through shared memory: the SL
    // step is MIO-throttled and staging costs an LDGSTS plus an LDS per node).
    // Plain SL rows up to 8192 nodes are double-buffered, so each step needs
    // one barrier (write the other buffer, sync, swap) instead of two.
    constexpr bool DBUF = KIND == MGRIT_KIND_SL && NPT <= 8;
    constexpr bool PREFETCH = NPT <= 8;
    const int n = L.n_x;
    const int m = A.m;
    RowCtx cx = make_ctx(sm, n, nbs, scratch, blockIdx.x, L, status);
    // layout after GmresSmem: [halo | rowB n | halo]
    double *const rowA = cx.rowbuf;
    double *const rowB = cx.bsm + kHalo;
    auto U = [&](int64_t t) { return A.U + (t - A.u_row0) * A.ldu; };
    auto Gr = [&](int64_t t) -> const double * { return A.G ? A.G + (t - A.g_row0) * A.ldg : nullptr; };
    auto Cb = [&](int64_t c) { return A.Cbuf + (c - A.c_row0) * (int64_t)n; };
    auto Ucr = [&](int64_t c) { return A.Uc + (c - A.c_row0) * (int64_t)n; };

    for (int64_t c = A.c_begin + blockIdx.x; c < A.c_begin + A.c_count; c += gridDim.x) {
        const int64_t t0 = c * m;
        const int64_t tC = t0 + m;
        double v[NPT], sv[NPT];
        load_records<NT, NPT, F>(L, t0, sv);
        // ---- left state of the interval
        const bool zero_left = A.zero_init && (c == 0 || A.phase == MGRIT_PHASE_FC ||
                                               A.phase == MGRIT_PHASE_FONLY_RES);
        if (zero_left) {
#pragma unroll
            for (int k = 0; k < NPT; ++k) v[k] = 0.0;
            if (c == 0 || A.phase == MGRIT_PHASE_FONLY_RES) store_row<NT, NPT, F>(U(t0), v, n);
        } else if (A.phase == MGRIT_PHASE_FC || A.phase == MGRIT_PHASE_FONLY_RES || c == 0) {
            load_row<NT, NPT, F>(v, U(t0), n);
        } else {
            load_row<NT, NPT, F>(v, Cb(c), n);
        }
        if (A.phase == MGRIT_PHASE_INJ_F) {
            // U[::m] += Uc  (mgrit.py:333)
            double u[NPT];
            load_row<NT, NPT, F>(u, Ucr(c), n);
#pragma unroll
            for (int k = 0; k < NPT; ++k) v[k] = __dadd_rn(v[k], u[k]);
            store_row<NT, NPT, F>(U(t0), v, n);
        } else if (A.phase == MGRIT_PHASE_F_RES && c > 0) {
            store_row<NT, NPT, F>(U(t0), v, n);
        }
        if constexpr (DBUF) cx.rowbuf = rowA;
        set_row<NT, NPT, F>(cx.rowbuf, v, n);

        // ---- F-relaxation chain (mgrit.py:276-283) then the interval tail at
        //      k == m; a single call site of the step operator keeps the
        //      kernel body (and its compile time) small.
        const bool last = (c + 1 == A.n_intervals);
        const int kmax = (A.phase == MGRIT_PHASE_INJ_F && !A.partial) ? m - 1 : m;
        if (A.phase == MGRIT_PHASE_INJ_F && !A.partial && last) {
            // U[N] += Uc[N/m] for the final C-point (mgrit.py:333)
            double right[NPT], u[NPT];
            load_row<NT, NPT, F>(right, Cb(c + 1), n);
            load_row<NT, NPT, F>(u, Ucr(c + 1), n);
#pragma unroll
            for (int k = 0; k < NPT; ++k) right[k] = __dadd_rn(right[k], u[k]);
            store_row<NT, NPT, F>(U(tC), right, n);
        }
#pragma unroll 1
        for (int k = 1; k <= kmax; ++k) {
            const int64_t t = t0 + k;
            double sn[PREFETCH ? NPT : 1];
            if constexpr (PREFETCH) {
                if (k < kmax) load_records<NT, NPT, F>(L, t, sn);
            }
            cta_apply<P, KIND, NT, NPT, F, false, (MINB > 1)>(L, t - 1, cx, v, sv);
            if constexpr (PREFETCH) {
#pragma unroll
                for (int q = 0; q < NPT; ++q) sv[q] = sn[q];
            } else {
                if (k < kmax) load_records<NT, NPT, F>(L, t, sv);
            }
            if (k < m) {
                add_forcing<NT, NPT, F>(v, Gr(t), n);
                store_row<NT, NPT, F>(U(t), v, n);
                if constexpr (DBUF) {
                    double *other = cx.rowbuf == rowB ? rowA : rowB;
#pragma unroll
                    for (int q = 0; q < NPT; ++q) {
                        const int i = threadIdx.x + q * NT;
                        if (F || i < n) put_row(other, i, v[q], n);
                    }
                    __syncthreads();
                    cx.rowbuf = other;
                } else {
                    set_row<NT, NPT, F>(cx.rowbuf, v, n);
                }
                continue;
            }
            // ---- interval tail at the right C-point tC = t
            if (A.phase == MGRIT_PHASE_FC) {
                // C-relaxation (mgrit.py:286-290) into the C-point buffer
                add_forcing<NT, NPT, F>(v, Gr(tC), n);
                store_row<NT, NPT, F>(Cb(c + 1), v, n);
                break;
            }
            // subtrahend of the C-point residual: the current U[tC]
            double right[NPT];
            if (A.phase == MGRIT_PHASE_INJ_F) {
                double u[NPT];
                load_row<NT, NPT, F>(right, Cb(c + 1), n);
                load_row<NT, NPT, F>(u, Ucr(c + 1), n);
#pragma unroll
                for (int q = 0; q < NPT; ++q) right[q] = __dadd_rn(right[q], u[q]);
                if (last) store_row<NT, NPT, F>(U(tC), right, n);
            } else if (A.phase == MGRIT_PHASE_F_RES) {
                load_row<NT, NPT, F>(right, Cb(c + 1), n);
                store_row<NT, NPT, F>(U(tC), right, n);
            } else {  // FONLY_RES
                if (A.zero_init) {
#pragma unroll
                    for (int q = 0; q < NPT; ++q) right[q] = 0.0;
                    store_row<NT, NPT, F>(U(tC), right, n);
                } else {
                    load_row<NT, NPT, F>(right, U(tC), n);
                }
                store_row<NT, NPT, F>(Cb(c + 1), right, n);
            }
            // r = (G + Phi U[tC-1]) - U[tC]; F-point residuals are exactly 0
            // after F-relaxation ((G + S) - (S + G) == 0 bitwise), so the
            // restriction Gc = R[::m] and the norm only need C-points.
            double ss = 0.0;
            const double *g = Gr(tC);
#pragma unroll
            for (int q = 0; q < NPT; ++q) {
                const int i = threadIdx.x + q * NT;
                if (F || i < n) {
                    const double r = __dsub_rn(__dadd_rn(g ? g[i] : 0.0, v[q]), right[q]);
                    v[q] = r;
                    ss = __dadd_rn(ss, __dmul_rn(r, r));
                }
            }
            if (A.Gc && A.phase != MGRIT_PHASE_INJ_F)
                store_row<NT, NPT, F>(A.Gc + (c + 1 - A.c_row0) * (int64_t)n, v, n);
            if (A.partial) {
                const double tot = block_sum2<NT>(ss, cx);
                if (threadIdx.x == 0) A.partial[c - A.partial0] = tot;
            }
        }
    }
}

// ---------------------------------------------------------------------------
// sequential sweep: one CTA steps the whole level

template <int P, int KIND, int NT, int NPT, bool F, bool NUMBA>
__global__ void __launch_bounds__(NT, 1) sweep_kernel(mgrit_level_desc L, double *U, int64_t ldu,
                                                   const double *G, int64_t ldg, int zero_init,
                                                   int32_t *gmres_iters, int nbs, double *scratch,
                                                   int32_t *status) {
    extern __shared__ double sm[];
    constexpr bool PREFETCH = NPT <= 8;
    const int n = L.n_x;
    RowCtx cx = make_ctx(sm, n, nbs, scratch, 0, L, status);
    double v[NPT], sv[NPT];
    load_records<NT, NPT, F>(L, 0, sv);
    if (zero_init) {
#pragma unroll
        for (int k = 0; k < NPT; ++k) v[k] = 0.0;
        store_row<NT, NPT, F>(U, v, n);
    } else {
        load_row<NT, NPT, F>(v, U, n);
    }
    set_row<NT, NPT, F>(cx.rowbuf, v, n);
#pragma unroll 1
    for (int64_t t = 0; t < L.n_steps; ++t) {
        double sn[PREFETCH ? NPT : 1];
        if constexpr (PREFETCH) {
            if (t + 1 < L.n_steps) load_records<NT, NPT, F>(L, t + 1, sn);
        }
        const int cnt = cta_apply<P, KIND, NT, NPT, F, NUMBA>(L, t, cx, v, sv);
        if constexpr (PREFETCH) {
#pragma unroll
            for (int q = 0; q < NPT; ++q) sv[q] = sn[q];
        } else {
            if (t + 1 < L.n_steps) load_records<NT, NPT, F>(L, t + 1, sv);
        }
        add_forcing<NT, NPT, F>(v, G ? G + (t + 1) * ldg : nullptr, n);
        store_row<NT, NPT, F>(U + (t + 1) * ldu, v, n);
        if (gmres_iters && threadIdx.x == 0) gmres_iters[t] = cnt;
        set_row<NT, NPT, F>(cx.rowbuf, v, n);
    }
}

// ---------------------------------------------------------------------------
// launch configuration: a CTA owns a whole row

struct Cfg1D {
    int nt, npt;
};

inline Cfg1D cfg_for(int n) {
    if (n <= 1024) return {256, 4};
    if (n <= 2048) return {512, 4};
    if (n <= 4096) return {1024, 4};
    if (n <= 8192) return {1024, 8};
    return {1024, 16};
}

inline int max_smem_optin() {
    int dev = 0, v = 48 * 1024;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    return v;
}

// Krylov slots that fit in shared memory next to the row
inline int smem_slots(const mgrit_level_desc *L) {
    // plain SL: second row buffer (its halo comes from the 2*kHalo spare
    // doubles smem_bytes_for always reserves)
    if (L->kind == MGRIT_KIND_SL) return L->n_x <= 8192 ? 1 : 0;
    if (L->kind != MGRIT_KIND_CORRECTED) return 0;
    const int64_t base = (int64_t)smem_bytes_for(L->n_x, 0);
    const int64_t avail = (int64_t)max_smem_optin() - base - 1024;
    int64_t k = avail > 0 ? avail / ((int64_t)L->n_x * 8) : 0;
    if (k > L->gmres_max_iters + 1) k = L->gmres_max_iters + 1;
    return (int)(k < 0 ? 0 : k);
}

// Krylov slots that fit when two CTAs share an SM (half of the SM's shared
// memory each, less the per-CTA reservation)
inline int smem_slots_two(const mgrit_level_desc *L) {
    int dev = 0, per_sm = 228 * 1024;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&per_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
    const int64_t avail = per_sm / 2 - 1024 - (int64_t)smem_bytes_for(L->n_x, 0);
    int64_t k = avail > 0 ? avail / ((int64_t)L->n_x * 8) : 0;
    if (k > L->gmres_max_iters + 1) k = L->gmres_max_iters + 1;
    return (int)(k < 0 ? 0 : k);
}

inline int resident_ctas(const void *fn, int nt, size_t smem) {
    int dev = 0, sms = 148, per = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fn, nt, smem) != cudaSuccess || per < 1)
        per = 1;
    return sms * per;
}

template <typename F>
inline int prep(F fn, size_t smem) {
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

template <int P_, int KIND_, int NT_, int NPT_, bool F_>
struct Tag {
    static constexpr int P = P_, KIND = KIND_, NT = NT_, NPT = NPT_;
    static constexpr bool F = F_;  // n == NT * NPT: no bounds checks
};

// corrected phases of 4096-node rows (256 threads x 16 nodes) also come in a
// two-CTAs-per-SM form (<= 128 registers, half the shared memory)
template <typename C>
struct TwoPerSM {
    static constexpr bool value = C::KIND == MGRIT_KIND_CORRECTED && C::NT == 256 && C::NPT == 16 && C::F;
};

// full rows (n == NT*NPT: the power-of-two meshes of every BASELINE config)
// compile without bounds checks; any other n uses a checked variant.
// Plain SL / forward-Euler steps are HBM/issue bound: 1024 threads x 4 nodes
// keep the most loads in flight.  Corrected (GMRES) steps are bound by the
// latency of ~K^2/2 dependent block reductions whose instruction cost scales
// with the warp count: 256 threads x n/256 nodes minimise it.
template <int P, int KIND, typename Fn>
static int dispatch_cfg(Cfg1D, int n, Fn &&f) {
    if constexpr (KIND == MGRIT_KIND_CORRECTED) {
        if (n == 1024) return f(Tag<P, KIND, 256, 4, true>{});
        if (n == 2048) return f(Tag<P, KIND, 256, 8, true>{});
        if (n == 4096) return f(Tag<P, KIND, 256, 16, true>{});
        if (n == 8192) return f(Tag<P, KIND, 512, 16, true>{});
        if (n == 16384) return f(Tag<P, KIND, 1024, 16, true>{});
    } else {
        if (n == 1024) return f(Tag<P, KIND, 256, 4, true>{});
        if (n == 2048) return f(Tag<P, KIND, 256, 8, true>{});
        if (n == 4096) return f(Tag<P, KIND, 1024, 4, true>{});
        if (n == 8192) return f(Tag<P, KIND, 1024, 8, true>{});
        if (n == 16384) return f(Tag<P, KIND, 1024, 16, true>{});
    }
    if (n < 1024) return f(Tag<P, KIND, 256, 4, false>{});
    return f(Tag<P, KIND, 1024, 16, false>{});
}

inline int validate(const mgrit_level_desc *L) {
    if (!L || L->dim != 1 || L->n_x < 8 || L->n_x > 16384 || !L->s_x) return MGRIT_EINVAL;
    if (L->p != 1 && L->p != 3 && L->p != 5) return MGRIT_EINVAL;
    if (L->kind < 0 || L->kind > 2) return MGRIT_EINVAL;
    if (L->kind != MGRIT_KIND_SL && !L->sig_x) return MGRIT_EINVAL;
    if (L->kind == MGRIT_KIND_CORRECTED && (L->gmres_max_iters < 1 || L->gmres_max_iters > kMaxKrylov))
        return MGRIT_EINVAL;
    return MGRIT_OK;
}

// global Krylov bytes one CTA needs beyond its shared-memory slots
inline int64_t scratch_per_cta(const mgrit_level_desc *L) {
    if (L->kind != MGRIT_KIND_CORRECTED) return 0;
    const int spill = L->gmres_max_iters + 1 - smem_slots(L);
    return spill > 0 ? (int64_t)spill * L->n_x * 8 : 0;
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
    static int64_t capacity(const mgrit_level_desc *L, bool one_per_sm);
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
int64_t Launch1D<P, KIND>::capacity(const mgrit_level_desc *L, bool one_per_sm) {
    const Cfg1D c = cfg_for(L->n_x);
    const int nbs = smem_slots(L);
    const size_t smem = smem_bytes_for(L->n_x, nbs);
    return dispatch_cfg<P, KIND>(c, L->n_x, [&](auto T) {
        using C = decltype(T);
        auto fn = rows_kernel<C::P, C::KIND, C::NT, C::NPT, C::F>;
        if (prep(fn, smem)) return 1;
        int cap = resident_ctas((const void *)fn, C::NT, smem);
        if constexpr (TwoPerSM<C>::value) {
            if (one_per_sm) return cap;
            // the phase kernel's two-CTAs-per-SM form (scratch is sized from this)
            const size_t smem2 = smem_bytes_for(L->n_x, smem_slots_two(L));
            auto fn2 = phase_kernel<C::P, C::KIND, C::NT, C::NPT, C::F, 2>;
            if (!prep(fn2, smem2)) {
                const int cap2 = resident_ctas((const void *)fn2, C::NT, smem2);
                if (cap2 > cap) cap = cap2;
            }
        }
        return cap;
    });
}

template <int P, int KIND>
int Launch1D<P, KIND>::rows(const mgrit_level_desc *L, const RowsArgs &a, void *scratch,
                            int64_t scratch_bytes, int32_t *status, cudaStream_t st) {
    int rc = validate(L);
    if (rc) return rc;
    if (a.B <= 0) return MGRIT_OK;
    const Cfg1D c = cfg_for(L->n_x);
    const int nbs = smem_slots(L);
    const size_t smem = smem_bytes_for(L->n_x, nbs);
    rc = dispatch_cfg<P, KIND>(c, L->n_x, [&](auto T) {
        using C = decltype(T);
        auto fn = rows_kernel<C::P, C::KIND, C::NT, C::NPT, C::F>;
        int r = prep(fn, smem);
        if (r) return r;
        const int grid = cap_grid(a.B, resident_ctas((const void *)fn, C::NT, smem), L, scratch_bytes);
        if (grid < 1) return (int)MGRIT_EINVAL;
        fn<<<grid, C::NT, smem, st>>>(*L, a, nbs, (double *)scratch, status);
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
    const int nbs = smem_slots(L);
    const size_t smem = smem_bytes_for(L->n_x, nbs);
    rc = dispatch_cfg<P, KIND>(c, L->n_x, [&](auto T) {
        using C = decltype(T);
        auto fn = phase_kernel<C::P, C::KIND, C::NT, C::NPT, C::F>;
        int r = prep(fn, smem);
        if (r) return r;
        const int res1 = resident_ctas((const void *)fn, C::NT, smem);
        if constexpr (TwoPerSM<C>::value) {
            // more row chains than SMs: two CTAs per SM (fewer shared-memory
            // Krylov slots, sigma re-read from L1) finish them in one wave
            // instead of two; the chains are latency bound, so two per SM
            // overlap their reduction chains
            if (A->c_count > res1 && L->launch_policy != MGRIT_LAUNCH_AUTO_ONE) {
                const int nbs2 = smem_slots_two(L);
                const size_t smem2 = smem_bytes_for(L->n_x, nbs2);
                auto fn2 = phase_kernel<C::P, C::KIND, C::NT, C::NPT, C::F, 2>;
                if ((r = prep(fn2, smem2))) return r;
                int64_t g = A->c_count;
                const int res2 = resident_ctas((const void *)fn2, C::NT, smem2);
                if (g > res2) g = res2;
                const int spill = L->gmres_max_iters + 1 - nbs2;
                const int64_t per = spill > 0 ? (int64_t)spill * L->n_x * 8 : 0;
                if (per > 0 && scratch_bytes / per < g) g = scratch_bytes / per;
                if (g > res1) {
                    fn2<<<(int)g, C::NT, smem2, st>>>(*L, *A, nbs2, (double *)scratch, status);
                    return (int)MGRIT_OK;
                }
            }
        }
        const int grid = cap_grid(A->c_count, res1, L, scratch_bytes);
        if (grid < 1) return (int)MGRIT_EINVAL;
        fn<<<grid, C::NT, smem, st>>>(*L, *A, nbs, (double *)scratch, status);
        return (int)MGRIT_OK;
    });
    if (rc) return rc;
    return check_launch("level_phase");
}

template <int P, int KIND>
int Launch1D<P, KIND>::sweep(const mgrit_level_desc *L, double *U, int64_t ldu, const double *G,
                             int64_t ldg, int zero_init, int32_t *gmres_iters, void *scratch,
                             int64_t scratch_bytes, int32_t *status, cudaStream_t st) {
    int rc = validate(L);
    if (rc) return rc;
    if (!U) return MGRIT_EINVAL;
    if (scratch_per_cta(L) > scratch_bytes) return MGRIT_EINVAL;
    const Cfg1D c = cfg_for(L->n_x);
    const int nbs = smem_slots(L);
    const size_t smem = smem_bytes_for(L->n_x, nbs);
    const bool numba = L->stencil_numba && L->kind == MGRIT_KIND_CORRECTED;
    rc = dispatch_cfg<P, KIND>(c, L->n_x, [&](auto T) {
        using C = decltype(T);
        int r;
        if constexpr (C::KIND == MGRIT_KIND_CORRECTED) {
            if (numba) {
                auto fn = sweep_kernel<C::P, C::KIND, C::NT, C::NPT, C::F, true>;
                if ((r = prep(fn, smem))) return r;
                fn<<<1, C::NT, smem, st>>>(*L, U, ldu, G, ldg, zero_init, gmres_iters, nbs, (double *)scratch,
                                           status);
                return (int)MGRIT_OK;
            }
        }
        auto fn = sweep_kernel<C::P, C::KIND, C::NT, C::NPT, C::F, false>;
        if ((r = prep(fn, smem))) return r;
        fn<<<1, C::NT, smem, st>>>(*L, U, ldu, G, ldg, zero_init, gmres_iters, nbs, (double *)scratch, status);
        return (int)MGRIT_OK;
    });
    if (rc) return rc;
    return check_launch("sequential_sweep");
}

#endif  // MGRIT_LAUNCH1D_IMPL

}  // namespace mgrit
