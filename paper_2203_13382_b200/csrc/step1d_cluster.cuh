// step1d_cluster.cuh — corrected coarse steps (SL + MGS-GMRES on
// I - diag(sigma) D, coarse_correction.py:173-240) with one thread-block
// CLUSTER of CS CTAs per row chain instead of one CTA.
//
// Why: a coarse level has few C-intervals (cfg2: 16, 4, 1 row chains on its
// three coarsest levels), so the one-CTA-per-chain kernel leaves >90% of the
// 148 SMs idle and every Arnoldi step is bound by one SM's shared-memory
// bandwidth (a 32 KB basis vector per projection) plus a block reduction.
// Splitting the row over a CS-CTA cluster (CS = 2, 4, 8 or 16, picked per
// level from measured costs, step1d_cl.cu) gives each SM an n/CS-node chunk
// (512 nodes at n = 4096, CS = 8); reductions become cluster all-reduces over
// DSMEM:
//   * every CTA reduces its partials, st.async-pushes them into every peer's
//     receive slot (mbarrier complete_tx), waits on its own mbarrier and sums
//     the CS contributions in rank order -> bit-identical totals in all CTAs,
//     so all CTAs run the same Arnoldi/Givens arithmetic in lock-step;
//   * the stencil halo (RAD <= 3 nodes each side) rides along with the norm
//     reduction: neighbours push their un-normalised edge values and every CTA
//     normalises them with the same division as the owner (bitwise equal);
//   * the full state row that the semi-Lagrangian gather needs is assembled
//     in every CTA by TMA multicast: each CTA bulk-copies its own freshly
//     stored chunk from global memory (L2) to the same offset in all CS CTAs.
// Everything except the order of the fp64 inner-product sums is the
// arithmetic of the one-CTA kernel (step1d_kernels.cuh cta_apply).
#pragma once
#include "step1d_kernels.cuh"

namespace mgrit {
namespace cl {

// CS (CTAs per cluster: 2, 4, 8 portable; 16 non-portable) is a template
// parameter of everything below; the launch policy picks it per level.
constexpr int NTC = 128;       // threads per CTA
constexpr int NWC = NTC / 32;  // warps per CTA
constexpr int kNV = 32;        // values of one fused multi-reduction (d_0..15, gram_0..15)
constexpr int kMaxKrylovCl = 10;  // Arnoldi steps unrolled at compile time (GmresConfig.max_iters)

// ---------------------------------------------------------------- PTX ----
__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t ctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t mapa(uint32_t a, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
    return r;
}
__device__ __forceinline__ void mbar_init(uint64_t *b, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *b, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "W%=:\n\tmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
        "\t@!p bra W%=;\n}" ::"r"(su32(b)),
        "r"(parity)
        : "memory");
}
// remote 8 / 16 byte store into a peer's shared memory, completing tx bytes
// on the peer's mbarrier
__device__ __forceinline__ void st_async1(uint32_t raddr, double v, uint32_t rbar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(raddr),
                 "l"(__double_as_longlong(v)), "r"(rbar)
                 : "memory");
}
__device__ __forceinline__ void st_async2(uint32_t raddr, double a, double b, uint32_t rbar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.b64 [%0], {%1, %2}, [%3];" ::"r"(raddr),
                 "l"(__double_as_longlong(a)), "l"(__double_as_longlong(b)), "r"(rbar)
                 : "memory");
}
__device__ __forceinline__ void fence_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }
// TMA bulk copy global -> the same smem offset in every CTA of `mask`
__device__ __forceinline__ void bulk_multicast(uint32_t dst, const void *src, uint32_t bytes, uint32_t bar,
                                               uint16_t mask) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1], %2, [%3], "
        "%4;" ::"r"(dst),
        "l"(src), "r"(bytes), "r"(bar), "h"(mask)
        : "memory");
}

// ------------------------------------------------------- shared memory ----
template <int CS>
struct __align__(16) ClSmem {
    uint64_t rbar[2];   // receive mbarriers, used alternately by successive reductions
    uint64_t rowbar;    // full-row arrival (TMA multicast)
    uint64_t pad_;
    double recv[2][CS * kNV];      // multi: [src rank][q]; single: [src rank * NWC + warp][2]
    double halo[2][2][kHalo];      // [buf][0: from rank-1 (left halo), 1: from rank+1 (right)]
    double wpart[NWC][kNV];        // per-warp partials of a multi-reduction
    double wred[2][NWC][2];        // per-warp partials of a scalar all-reduce
    double H[(kMaxKrylov + 1) * kMaxKrylov];
    double cs[kMaxKrylov], sn[kMaxKrylov], g[kMaxKrylov + 1], y[kMaxKrylov];
    double gram[kMaxKrylov * kMaxKrylov];
    double hv[kMaxKrylov];
    double rdiag[kMaxKrylov];  // RN(1 / H_jj), shared by the rotation and the back substitution
    int stop;
};

template <int CS>
struct ClCtx {
    ClSmem<CS> *S;
    double *row;     // full state row (global node index), halo kHalo each side
    const double *grow;  // GG (rows too large for shared memory): the global row
    bool zrow;           // GG: the current row is all zeros
    double *slots;   // Krylov chunks: slot j interior at slots + j*ld + kHalo
    int ld;          // chunk + 2*kHalo
    int n, chunk;
    uint32_t rank, base;
    uint32_t seq;    // reductions issued so far (buffer = seq & 1)
    uint32_t pubs;   // row publications consumed so far
    int32_t *status;
    __device__ double *slot(int j) const { return slots + j * ld + kHalo; }
};

// GG ("global gather"): rows too large for a shared-memory copy next to the
// Krylov chunks (n = 16384 at CS = 8 or 16) are gathered straight from L2;
// publication is then a cluster barrier (release / acquire) instead of a TMA
// multicast.
// (decided for the largest Krylov space, kMaxKrylovCl + 1 chunk slots)
constexpr size_t kClSmemMax = 227 * 1024;
template <int CS>
__host__ __device__ constexpr bool cl_gg(int n) {
    return sizeof(ClSmem<CS>) + sizeof(double) * ((size_t)n + 2 * kHalo) +
               sizeof(double) * (size_t)(kMaxKrylovCl + 1) * (n / CS + 2 * kHalo) > kClSmemMax;
}

template <int CS>
__host__ __device__ inline size_t cl_smem_bytes(int n, int K) {
    const int chunk = n / CS;
    return sizeof(ClSmem<CS>) + (cl_gg<CS>(n) ? 0 : sizeof(double) * ((size_t)n + 2 * kHalo)) +
           sizeof(double) * (size_t)(K + 1) * (chunk + 2 * kHalo);
}

template <int CS>
__device__ __forceinline__ ClCtx<CS> make_clctx(int n, int K, int32_t *status) {
    extern __shared__ __align__(128) unsigned char clsm[];
    ClCtx<CS> c;
    c.S = reinterpret_cast<ClSmem<CS> *>(clsm);
    c.row = reinterpret_cast<double *>(clsm + sizeof(ClSmem<CS>)) + kHalo;
    c.grow = nullptr;
    c.zrow = false;
    c.chunk = n / CS;
    c.ld = c.chunk + 2 * kHalo;
    c.slots = cl_gg<CS>(n) ? c.row - kHalo : c.row + n + kHalo;
    c.n = n;
    c.rank = ctarank();
    c.base = c.rank * c.chunk;
    c.seq = 0;
    c.pubs = 0;
    c.status = status;
    (void)K;
    return c;
}

// ----------------------------------------------------- cluster reductions --
// All-reduce of one (TWO: two) scalars, split into send / receive so the
// caller can overlap independent work with the DSMEM round trip.  Warp
// butterflies, one barrier, then lanes 0..CS-1 of warp 0 each sum the NWC
// warp partials and push the CTA total to one peer; the receiver sums the CS
// totals in rank order (bit-identical in all CTAs).  With EDGES the CTA's
// first / last RAD chunk values (v[0] of threads < RAD, v[NPT-1] of threads
// >= NTC-RAD) go to the neighbours' halo slots.
struct ArTok {
    uint32_t buf, par;
};

template <int NPT, int RAD, bool EDGES, bool TWO, int CS>
__device__ __forceinline__ ArTok ar_send(ClCtx<CS> &cx, double a, double b, const double (&v)[NPT], int pid = -1) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    ClSmem<CS> &S = *cx.S;
    const ArTok tk{cx.seq & 1, (cx.seq >> 1) & 1};
    ++cx.seq;
    if (pid >= 0) MGRIT_PROBE_AT(pid);
    const uint32_t lbar = su32(&S.rbar[tk.buf]);
    if constexpr (EDGES) {
        if (tid < RAD) {
            const uint32_t peer = (cx.rank + CS - 1) % CS;
            st_async1(mapa(su32(&S.halo[tk.buf][1][tid]), peer), v[0], mapa(lbar, peer));
        }
        if (tid >= NTC - RAD) {
            const uint32_t peer = (cx.rank + 1) % CS;
            st_async1(mapa(su32(&S.halo[tk.buf][0][tid - (NTC - RAD)]), peer), v[NPT - 1], mapa(lbar, peer));
        }
    }
    a = warp_sum(a);
    if constexpr (TWO) b = warp_sum(b);
    if (lane == 0) {
        S.wred[tk.buf][warp][0] = a;
        if constexpr (TWO) S.wred[tk.buf][warp][1] = b;
    }
    __syncthreads();
    if (pid >= 0) MGRIT_PROBE_AT(pid + 1);
    if (warp == 0) {
        if (lane == 0) mbar_expect_tx(&S.rbar[tk.buf], CS * (TWO ? 16 : 8) + (EDGES ? 2 * RAD * 8 : 0));
        if (lane < CS) {
            double pa[NWC], pb[NWC] = {};
#pragma unroll
            for (int w = 0; w < NWC; ++w) {
                pa[w] = S.wred[tk.buf][w][0];
                pb[w] = TWO ? S.wred[tk.buf][w][1] : 0.0;
            }
#pragma unroll
            for (int w = 1; w < NWC; w <<= 1)
#pragma unroll
                for (int s = 0; s + w < NWC; s += 2 * w) {
                    pa[s] = __dadd_rn(pa[s], pa[s + w]);
                    if constexpr (TWO) pb[s] = __dadd_rn(pb[s], pb[s + w]);
                }
            if constexpr (TWO) {
                st_async2(mapa(su32(&S.recv[tk.buf][2 * cx.rank]), lane), pa[0], pb[0], mapa(lbar, lane));
            } else {
                st_async1(mapa(su32(&S.recv[tk.buf][cx.rank]), lane), pa[0], mapa(lbar, lane));
            }
        }
    }
    if (pid >= 0) MGRIT_PROBE_AT(pid + 2);
    return tk;
}

template <bool TWO, int CS>
__device__ __forceinline__ double2 ar_recv(ClCtx<CS> &cx, ArTok tk, int pid = -1) {
    ClSmem<CS> &S = *cx.S;
    mbar_wait(&S.rbar[tk.buf], tk.par);
    if (pid >= 0) MGRIT_PROBE_AT(pid + 3);
    const double *r = S.recv[tk.buf];
    double sa[CS], sb[TWO ? CS : 1];
#pragma unroll
    for (int s = 0; s < CS; ++s) {
        sa[s] = r[TWO ? 2 * s : s];
        if constexpr (TWO) sb[s] = r[2 * s + 1];
    }
#pragma unroll
    for (int w = 1; w < CS; w <<= 1)
#pragma unroll
        for (int s = 0; s + w < CS; s += 2 * w) {
            sa[s] = __dadd_rn(sa[s], sa[s + w]);
            if constexpr (TWO) sb[s] = __dadd_rn(sb[s], sb[s + w]);
        }
    if (pid >= 0) MGRIT_PROBE_AT(pid + 4);
    return make_double2(sa[0], TWO ? sb[0] : 0.0);
}

// Fused multi-reduction of x[0..V): warp 0 lane q (< NV) returns the cluster
// total of value q.  Intra-warp: recursive-halving transpose (V-1 shuffles,
// plus log2(32/V) butterfly levels), one barrier, warp 0 sums the NWC warp
// partials and pushes value q to every peer; the receiver sums the CS CTA
// totals in rank order.
template <int V, int NV, int CS>
__device__ __forceinline__ double ar_multi(ClCtx<CS> &cx, double (&x)[V]) {
    static_assert(V == 16 || V == 32, "V");
    static_assert(NV <= V, "NV");
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    ClSmem<CS> &S = *cx.S;
    const uint32_t buf = cx.seq & 1, par = (cx.seq >> 1) & 1;
    ++cx.seq;
#pragma unroll
    for (int s = V / 2; s >= 1; s >>= 1) {
        const bool upper = (lane & s) != 0;
#pragma unroll
        for (int i = 0; i < s; ++i) {
            const double send = upper ? x[i] : x[i + s];
            const double keep = upper ? x[i + s] : x[i];
            x[i] = __dadd_rn(keep, __shfl_xor_sync(0xffffffffu, send, s));
        }
    }
#pragma unroll
    for (int s = V; s < 32; s <<= 1) x[0] = __dadd_rn(x[0], __shfl_xor_sync(0xffffffffu, x[0], s));
    S.wpart[warp][lane] = x[0];
    __syncthreads();
    double tot = 0.0;
    if (warp == 0) {
        double p[NWC];
#pragma unroll
        for (int w = 0; w < NWC; ++w) p[w] = S.wpart[w][lane];
#pragma unroll
        for (int w = 1; w < NWC; w <<= 1)
#pragma unroll
            for (int s = 0; s + w < NWC; s += 2 * w) p[s] = __dadd_rn(p[s], p[s + w]);
        const uint32_t lbar = su32(&S.rbar[buf]);
        if (lane == 0) mbar_expect_tx(&S.rbar[buf], CS * NV * 8);
        if (lane < NV) {
            const uint32_t dst = su32(&S.recv[buf][cx.rank * kNV + lane]);
#pragma unroll
            for (int q = 0; q < CS; ++q) st_async1(mapa(dst, q), p[0], mapa(lbar, q));
        }
        mbar_wait(&S.rbar[buf], par);
        double t[CS];
#pragma unroll
        for (int s = 0; s < CS; ++s) t[s] = S.recv[buf][s * kNV + lane];
#pragma unroll
        for (int w = 1; w < CS; w <<= 1)
#pragma unroll
            for (int s = 0; s + w < CS; s += 2 * w) t[s] = __dadd_rn(t[s], t[s + w]);
        tot = t[0];
    }
    return tot;
}

// ------------------------------------------------------- row publication --
// Every CTA multicasts its own chunk of `src` (a global row it has stored, or
// that an earlier kernel wrote) into the full-row buffer of all CTAs; rank 0
// and rank CS-1 also supply the periodic halos.  GG: the chunk stores are
// released with a cluster-barrier arrive; await_row is the acquire wait.
template <bool GG, int CS>
__device__ __forceinline__ void publish_row(ClCtx<CS> &cx, const double *src) {
    if constexpr (GG) {
        asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
        cx.grow = src;
        cx.zrow = false;
        return;
    }
    fence_async_global();
    __syncthreads();
    if (threadIdx.x == 0) {
        ClSmem<CS> &S = *cx.S;
        const uint32_t bar = su32(&S.rowbar);
        const uint16_t mask = (uint16_t)((1u << CS) - 1);
        mbar_expect_tx(&S.rowbar, (uint32_t)((cx.n + 2 * kHalo) * 8));
        bulk_multicast(su32(cx.row + cx.base), src + cx.base, (uint32_t)(cx.chunk * 8), bar, mask);
        if (cx.rank == 0) bulk_multicast(su32(cx.row + cx.n), src, kHalo * 8, bar, mask);
        if (cx.rank == CS - 1) bulk_multicast(su32(cx.row - kHalo), src + cx.n - kHalo, kHalo * 8, bar, mask);
    }
}
template <bool GG, int CS>
__device__ __forceinline__ void await_row(ClCtx<CS> &cx) {
    if constexpr (GG) {
        asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
        return;
    }
    mbar_wait(&cx.S->rowbar, cx.pubs & 1);
    ++cx.pubs;
}
// local all-zero row (no publication)
template <bool GG, int CS>
__device__ __forceinline__ void zero_row(ClCtx<CS> &cx) {
    if constexpr (GG) {
        cx.zrow = true;
        return;
    }
    __syncthreads();
    for (int i = threadIdx.x - kHalo; i < cx.n + kHalo; i += NTC) cx.row[i] = 0.0;
    __syncthreads();
}

template <int NPT, int CS>
__device__ __forceinline__ void load_chunk(const ClCtx<CS> &cx, double (&v)[NPT], const double *src) {
#pragma unroll
    for (int k = 0; k < NPT; ++k) v[k] = src[cx.base + threadIdx.x + k * NTC];
}
template <int NPT, int CS>
__device__ __forceinline__ void store_chunk(const ClCtx<CS> &cx, double *dst, const double (&v)[NPT]) {
#pragma unroll
    for (int k = 0; k < NPT; ++k) dst[cx.base + threadIdx.x + k * NTC] = v[k];
}
template <int NPT, int CS>
__device__ __forceinline__ void add_forcing_chunk(const ClCtx<CS> &cx, double (&v)[NPT], const double *g) {
#pragma unroll
    for (int k = 0; k < NPT; ++k) v[k] = __dadd_rn(v[k], g ? g[cx.base + threadIdx.x + k * NTC] : 0.0);
}
template <int NPT, int CS>
__device__ __forceinline__ void load_records_chunk(const ClCtx<CS> &cx, const mgrit_level_desc &L, int64_t t,
                                                   double (&sv)[NPT]) {
    const double *s = L.s_x + (L.shared ? 0 : t) * (int64_t)cx.n + cx.base;
#pragma unroll
    for (int k = 0; k < NPT; ++k) sv[k] = __ldg(s + threadIdx.x + k * NTC);
}

// -------------------------------------------------- one corrected step ----
// Arnoldi steps are unrolled at compile time (kMaxKrylovCl = the reference's
// GmresConfig.max_iters); every thread keeps the Givens rotations in
// registers and evaluates them redundantly (identical inputs -> identical
// results in every thread and CTA), so the stop test needs no barrier.

// v (chunk) = Phi_t(row): SL gather from the full row, then GMRES on
// (I - diag(sig) D) x = v with the cluster reductions above.  Returns the
// Arnoldi count (-1 on a non-finite right-hand side).
template <int P, int NPT, bool NUMBA, bool LOWSYNC, bool GG, int CS>
__device__ int cl_apply(const mgrit_level_desc &L, int64_t t, ClCtx<CS> &cx, double (&v)[NPT],
                        const double (&sv)[NPT], bool wait_row) {
    constexpr int SLW = Stencil<P>::L;
    constexpr int RAD = (P + 1) / 2;
    constexpr int KM = kMaxKrylovCl;
    const int n = cx.n, tid = threadIdx.x;
    ClSmem<CS> &S = *cx.S;
    // ---- semi-Lagrangian gather (same arithmetic as cta_apply)
    MGRIT_PROBE_AT(400);
    if (wait_row) await_row<GG>(cx);
    MGRIT_PROBE_AT(401);
#pragma unroll
    for (int k = 0; k < NPT; ++k) {
        const Dec d = decompose_s(sv[k], n);
        double w[P + 1];
        lagrange_weights<P>(d.eps, w);
        double tap[P + 1];
        if constexpr (GG) {
            // periodic taps straight from the (L2-resident) global row
#pragma unroll
            for (int c = 0; c <= P; ++c) {
                int idx = d.e - SLW + c;
                idx += idx < 0 ? n : 0;
                idx -= idx >= n ? n : 0;
                tap[c] = cx.zrow ? 0.0 : __ldcg(cx.grow + idx);
            }
        } else {
            const double *src = cx.row + (d.e - SLW);
#pragma unroll
            for (int c = 0; c <= P; ++c) tap[c] = src[c];
        }
        double acc = 0.0;
#pragma unroll
        for (int c = 0; c <= P; ++c) {
            const double prod = __dmul_rn(tap[c], w[c]);
            acc = c == 0 ? prod : __dadd_rn(acc, prod);
        }
        v[k] = acc;
    }
    if (L.kind == MGRIT_KIND_SL) {
        // plain SL step (the cluster-split sequential sweep of a fine level):
        // no solve.  Every CTA must be done reading the shared-memory row
        // before anyone's publish_row multicasts the next one into it.
        if constexpr (!GG) cluster_sync_all();
        return 0;
    }
    const int64_t set = L.shared ? 0 : t;
    const double *sig = L.sig_x + set * (int64_t)n + cx.base;
    // sigma in registers, or re-read (L1) for the widest rows
    constexpr bool SGREG = NPT <= 8;
    double sg[SGREG ? NPT : 1];
    if constexpr (SGREG) {
#pragma unroll
        for (int k = 0; k < NPT; ++k) sg[k] = __ldg(sig + tid + k * NTC);
    }
    // (I - diag(sig) D) x at local node li on slot buffer b
    auto imsd_at = [&](const double *b, int k, int li, double xi) -> double {
        double acc;
        if constexpr (NUMBA) {
            acc = 0.0;
#pragma unroll
            for (int q = -RAD; q <= RAD; ++q) acc = __dadd_rn(acc, cmul<P>(RAD + q, b[li + q]));
        } else {
            acc = cmul<P>(RAD, xi);
#pragma unroll
            for (int q = 1; q <= RAD; ++q)
                acc = __dadd_rn(acc, __dadd_rn(cmul<P>(RAD + q, b[li + q]), cmul<P>(RAD - q, b[li - q])));
        }
        double s_i;
        if constexpr (SGREG) s_i = sg[k];
        else s_i = __ldg(sig + li);
        return __dsub_rn(xi, __dmul_rn(s_i, acc));
    };
    auto sumsq = [&]() -> double {
        double a = 0.0;
#pragma unroll
        for (int k = 0; k < NPT; ++k) a = fma(v[k], v[k], a);
        return a;
    };
    // write a normalised vector into slot j: interior from registers, halos
    // from the neighbours' pushed edge values divided the same way
    auto put_slot = [&](int j, double den, double rden, uint32_t hbuf) {
        double *b = cx.slot(j);
#pragma unroll
        for (int k = 0; k < NPT; ++k) b[tid + k * NTC] = v[k];
        if (tid < RAD) b[tid - RAD] = div_rcp(S.halo[hbuf][0][tid], den, rden);
        else if (tid < 2 * RAD) b[cx.chunk + tid - RAD] = div_rcp(S.halo[hbuf][1][tid - RAD], den, rden);
    };

    const int K = L.gmres_max_iters;
    const double tol = L.gmres_tol;
    MGRIT_PROBE_AT(402);
    int bad = 0;
#pragma unroll
    for (int k = 0; k < NPT; ++k)
        if (!isfinite(v[k])) bad = 1;
    const ArTok tb = ar_send<NPT, RAD, true, true>(cx, sumsq(), (double)bad, v);
    const double2 bs = ar_recv<true>(cx, tb);
    MGRIT_PROBE_AT(403);
    if (bs.y != 0.0) {
        if (tid == 0 && cx.rank == 0) atomicExch(cx.status, 1);
#pragma unroll
        for (int k = 0; k < NPT; ++k) v[k] = __longlong_as_double(0x7ff8000000000000LL);
        return -1;
    }
    const double beta = sqrt(bs.x);
    if (beta == 0.0) {
#pragma unroll
        for (int k = 0; k < NPT; ++k) v[k] = 0.0;
        return 0;
    }
    {
        const double yb = __drcp_rn(beta);
#pragma unroll
        for (int k = 0; k < NPT; ++k) v[k] = div_rcp(v[k], beta, yb);
        put_slot(0, beta, yb, tb.buf);
    }
    MGRIT_PROBE_AT(404);
    double cs[KM], sn[KM];  // Givens rotations (identical in every thread)
    double g_k = beta;
    double gmax = 0.0;      // warp 0: max |<b_i, b_j>|, i != j (low-sync)
    int done = 0;
    // The rotation of column kk (and the stop test it feeds) is applied after
    // the NEXT Arnoldi step's stencil: the two are independent, so the
    // rotation's dependent chain (hypot, reciprocal, divisions) overlaps the
    // stencil instead of following it.  If the test stops the iteration, that
    // stencil's result is discarded (it only wrote registers), so the
    // arithmetic and the step count are those of the reference's loop.
    double hprev = 0.0, nprev = 0.0;  // column kk-1: rotated H[kk-1][kk-1], h_{kk,kk-1}
    bool bprev = false, stopped = false;
    auto rotation = [&](int col, double hr, double nr, double &c_out, double &s_out) {
        const double den = hypot(hr, nr);
        const double rden = __drcp_rn(den);
        c_out = div_rcp(hr, den, rden);
        s_out = div_rcp(nr, den, rden);
        const double gn = __dmul_rn(-s_out, g_k);
        if (tid == 0) {
            S.H[col * kMaxKrylov + col] = den;
            S.rdiag[col] = rden;
            S.g[col] = __dmul_rn(c_out, g_k);
        }
        g_k = gn;
        done = col + 1;
        return fabs(gn) <= __dmul_rn(tol, beta);
    };
#pragma unroll
    for (int kk = 0; kk < KM; ++kk) {
        if (kk >= K) break;
        __syncthreads();  // slot kk complete (interior + halos)
        MGRIT_PROBE_AT(410 + 6 * kk);
        const double *bk = cx.slot(kk);
#pragma unroll
        for (int k = 0; k < NPT; ++k) v[k] = imsd_at(bk, k, tid + k * NTC, v[k]);
        if (kk > 0) {
            const bool conv = rotation(kk - 1, hprev, nprev, cs[kk - 1], sn[kk - 1]);
            if (bprev || (tol >= 0.0 && conv)) {
                stopped = true;
                break;
            }
        }
        MGRIT_PROBE_AT(411 + 6 * kk);
        double h[KM];
        if constexpr (LOWSYNC) {
            // one fused reduction of d_j = <b_j, w> (j <= kk) and the Gram
            // row <b_kk, b_i> (i < kk); the MGS coefficients follow from
            // h_j = d_j - sum_{i<j} G[j][i] h_i (exact in exact arithmetic)
            constexpr int V = 2 * KM + 1 > 16 ? 32 : 16;
            double x[V];
#pragma unroll
            for (int q = 0; q < V; ++q) x[q] = 0.0;
            double bkr[NPT];
#pragma unroll
            for (int k = 0; k < NPT; ++k) bkr[k] = bk[tid + k * NTC];
#pragma unroll
            for (int j = 0; j <= kk; ++j) {
                const double *bj = cx.slot(j);
#pragma unroll
                for (int k = 0; k < NPT; ++k) {
                    const double b = bj[tid + k * NTC];
                    x[j] = fma(b, v[k], x[j]);
                    if (j < kk) x[kk + 1 + j] = fma(b, bkr[k], x[kk + 1 + j]);
                }
            }
            const double tot = ar_multi<V, 2 * KM + 1>(cx, x);
            if (tid < 32) {
                const int lane = tid;
                const bool grow = lane > kk && lane <= 2 * kk;
                if (grow) S.gram[kk * kMaxKrylov + lane - kk - 1] = tot;
                double gm = grow ? fabs(tot) : 0.0;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) gm = fmax(gm, __shfl_xor_sync(0xffffffffu, gm, o));
                gmax = fmax(gmax, gm);
                __syncwarp();
                const double d = lane <= kk ? tot : 0.0;
                double hh = d;
                // Gram row of this lane (branch-free: clamped row, masked use)
                const double *grow_l = S.gram + (lane <= kk ? lane : 0) * kMaxKrylov;
                if (gmax <= 1e-9) {
                    // |G_ij| <= 1e-9: the second-order term of (I + L)^{-1} d
                    // is below 2.3e-16 |h| (|L| <= 15e-9), under the rounding
                    // of d itself -> first-order form, all shuffles independent
#pragma unroll
                    for (int i = 0; i < kk; ++i) {
                        const double di = __shfl_sync(0xffffffffu, d, i);
                        const double gi = grow_l[i];
                        hh = (i < lane && lane <= kk) ? fma(-gi, di, hh) : hh;
                    }
                } else {
#pragma unroll
                    for (int i = 0; i < kk; ++i) {
                        const double hi = __shfl_sync(0xffffffffu, hh, i);
                        const double gi = grow_l[i];
                        hh = (i < lane && lane <= kk) ? fma(-gi, hi, hh) : hh;
                    }
                }
                if (lane <= kk) S.hv[lane] = hh;
            }
            __syncthreads();
#pragma unroll
            for (int j = 0; j <= kk; ++j) h[j] = S.hv[j];
#pragma unroll
            for (int j = 0; j <= kk; ++j) {
                const double *bj = cx.slot(j);
#pragma unroll
                for (int k = 0; k < NPT; ++k) v[k] = fma(-h[j], bj[tid + k * NTC], v[k]);
            }
        } else {
            // modified Gram-Schmidt, one cluster all-reduce per projection
#pragma unroll
            for (int j = 0; j <= kk; ++j) {
                const double *bj = cx.slot(j);
                double bjr[NPT];
                double part = 0.0;
#pragma unroll
                for (int k = 0; k < NPT; ++k) {
                    bjr[k] = bj[tid + k * NTC];
                    part = fma(bjr[k], v[k], part);
                }
                const ArTok tk = ar_send<NPT, RAD, false, false>(cx, part, 0.0, v);
                h[j] = ar_recv<false>(cx, tk).x;
#pragma unroll
                for (int k = 0; k < NPT; ++k) v[k] = fma(-h[j], NPT <= 8 ? bjr[k] : bj[tid + k * NTC], v[k]);
            }
        }
        // norm of w (+ halo exchange of its edge values); the previous
        // rotations are applied to column kk while the partials are in flight
        MGRIT_PROBE_AT(412 + 6 * kk);
        const ArTok tn = ar_send<NPT, RAD, true, false>(cx, sumsq(), 0.0, v);
        double hrun = h[0];
#pragma unroll
        for (int j = 1; j <= kk; ++j) {
            const double tmp = __dadd_rn(__dmul_rn(cs[j - 1], hrun), __dmul_rn(sn[j - 1], h[j]));
            hrun = __dadd_rn(__dmul_rn(-sn[j - 1], hrun), __dmul_rn(cs[j - 1], h[j]));
            if (tid == 0) S.H[(j - 1) * kMaxKrylov + kk] = tmp;
        }
        const double nrm = sqrt(ar_recv<false>(cx, tn).x);
        MGRIT_PROBE_AT(413 + 6 * kk);
        const bool brk = nrm <= __dmul_rn(1e-14, beta);
        // b_{kk+1} = w / h_{kk+1,kk}; written even on breakdown (the slot is
        // then never read: the loop stops and x uses slots < kk + 1), so
        // the normalisation and the rotation below form one basic block
        // whose two dependent chains the scheduler can interleave
        {
            const double yn = __drcp_rn(nrm);
#pragma unroll
            for (int k = 0; k < NPT; ++k) v[k] = div_rcp(v[k], nrm, yn);
            put_slot(kk + 1, nrm, yn, tn.buf);
        }
        MGRIT_PROBE_AT(414 + 6 * kk);
        hprev = hrun;
        nprev = nrm;
        bprev = brk;
        MGRIT_PROBE_AT(415 + 6 * kk);
    }
    if (!stopped) {
        // the last column's rotation (the iteration ended at K steps)
        double c_last, s_last;
        rotation(K - 1, hprev, nprev, c_last, s_last);
    }
    __syncthreads();  // S.H / S.g / S.rdiag from thread 0
    MGRIT_PROBE_AT(482);
    // back substitution (warp 0; y_j = acc / H_jj via the stored reciprocal,
    // correctly rounded) and x = sum_j b_j y_j on the chunk
    if (tid < 32) {
        const int lane = tid;
        double acc = lane < done ? S.g[lane] : 0.0;
        const double hjj = lane < done ? S.H[lane * kMaxKrylov + lane] : 1.0;
        const double rjj = lane < done ? S.rdiag[lane] : 1.0;
        // steps j >= done are skipped (warp-uniform branch; y_j stays 0)
        double myy = 0.0;
#pragma unroll
        for (int j = KM - 1; j >= 0; --j) {
            if (j >= done) continue;
            const bool upd = lane < j;
            const double hlj = upd ? S.H[lane * kMaxKrylov + j] : 0.0;
            const double yj = __shfl_sync(0xffffffffu, div_rcp(acc, hjj, rjj), j);
            myy = lane == j ? yj : myy;
            acc = upd ? __dsub_rn(acc, __dmul_rn(hlj, yj)) : acc;
        }
        if (lane < KM) S.y[lane] = myy;
    }
    MGRIT_PROBE_AT(483);
    __syncthreads();
    MGRIT_PROBE_AT(484);
#pragma unroll
    for (int k = 0; k < NPT; ++k) v[k] = 0.0;
    // j ascending over the done slots (uniform bound across the cluster)
#pragma unroll
    for (int j = 0; j < KM; ++j) {
        if (j >= done) break;
        const double yj = S.y[j];
        const double *bj = cx.slot(j);
#pragma unroll
        for (int k = 0; k < NPT; ++k) v[k] = fma(bj[tid + k * NTC], yj, v[k]);
    }
    MGRIT_PROBE_AT(481);
    return done;
}

template <int CS>
__device__ __forceinline__ void cl_init(ClCtx<CS> &cx) {
    if (threadIdx.x == 0) {
        mbar_init(&cx.S->rbar[0], 1);
        mbar_init(&cx.S->rbar[1], 1);
        mbar_init(&cx.S->rowbar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    cluster_sync_all();
}

// --------------------------------------------------------- level phases --
// Same phase semantics as phase_kernel (mgrit_b200.h MGRIT_PHASE_*), one
// cluster per C-interval (persistent over intervals).
template <int P, int NPT, bool LOWSYNC, bool GG, int CS>
__global__ void __launch_bounds__(NTC) cl_phase_kernel(mgrit_level_desc L, mgrit_phase_args A, int32_t *status) {
    const int n = L.n_x;
    const int m = A.m;
    ClCtx<CS> cx = make_clctx<CS>(n, L.gmres_max_iters, status);
    cl_init(cx);
    auto U = [&](int64_t t) { return A.U + (t - A.u_row0) * A.ldu; };
    auto Gr = [&](int64_t t) -> const double * { return A.G ? A.G + (t - A.g_row0) * A.ldg : nullptr; };
    auto Cb = [&](int64_t c) { return A.Cbuf + (c - A.c_row0) * (int64_t)n; };
    auto Ucr = [&](int64_t c) { return A.Uc + (c - A.c_row0) * (int64_t)n; };
    const int64_t cid = blockIdx.x / CS, ncl = gridDim.x / CS;

    for (int64_t c = A.c_begin + cid; c < A.c_begin + A.c_count; c += ncl) {
        const int64_t t0 = c * m;
        const int64_t tC = t0 + m;
        double v[NPT], sv[NPT];
        load_records_chunk<NPT>(cx, L, t0, sv);
        const bool zero_left = A.zero_init && (c == 0 || A.phase == MGRIT_PHASE_FC ||
                                               A.phase == MGRIT_PHASE_FONLY_RES);
        const double *pub = nullptr;  // global row holding the left state, if any
        if (zero_left) {
#pragma unroll
            for (int k = 0; k < NPT; ++k) v[k] = 0.0;
            if (c == 0 || A.phase == MGRIT_PHASE_FONLY_RES) store_chunk<NPT>(cx, U(t0), v);
        } else if (A.phase == MGRIT_PHASE_FC || A.phase == MGRIT_PHASE_FONLY_RES || c == 0) {
            load_chunk<NPT>(cx, v, U(t0));
            pub = U(t0);
        } else {
            load_chunk<NPT>(cx, v, Cb(c));
            pub = Cb(c);
        }
        if (A.phase == MGRIT_PHASE_INJ_F) {
            double u[NPT];
            load_chunk<NPT>(cx, u, Ucr(c));
#pragma unroll
            for (int k = 0; k < NPT; ++k) v[k] = __dadd_rn(v[k], u[k]);
            store_chunk<NPT>(cx, U(t0), v);
            pub = U(t0);
        } else if (A.phase == MGRIT_PHASE_F_RES && c > 0) {
            store_chunk<NPT>(cx, U(t0), v);
        }
        if (pub) publish_row<GG>(cx, pub);
        else zero_row<GG>(cx);  // local, nothing to wait for
        bool have_pub = pub != nullptr;

        const bool last = (c + 1 == A.n_intervals);
        const int kmax = (A.phase == MGRIT_PHASE_INJ_F && !A.partial) ? m - 1 : m;
        if (A.phase == MGRIT_PHASE_INJ_F && !A.partial && last) {
            double right[NPT], u[NPT];
            load_chunk<NPT>(cx, right, Cb(c + 1));
            load_chunk<NPT>(cx, u, Ucr(c + 1));
#pragma unroll
            for (int k = 0; k < NPT; ++k) right[k] = __dadd_rn(right[k], u[k]);
            store_chunk<NPT>(cx, U(tC), right);
        }
#pragma unroll 1
        for (int k = 1; k <= kmax; ++k) {
            const int64_t t = t0 + k;
            cl_apply<P, NPT, false, LOWSYNC, GG, CS>(L, t - 1, cx, v, sv, have_pub);
            have_pub = true;
            if (k < kmax) load_records_chunk<NPT>(cx, L, t, sv);
            if (k < m) {
                add_forcing_chunk<NPT>(cx, v, Gr(t));
                store_chunk<NPT>(cx, U(t), v);
                if (k < kmax) publish_row<GG>(cx, U(t));
                continue;
            }
            if (A.phase == MGRIT_PHASE_FC) {
                add_forcing_chunk<NPT>(cx, v, Gr(tC));
                store_chunk<NPT>(cx, Cb(c + 1), v);
                break;
            }
            double right[NPT];
            if (A.phase == MGRIT_PHASE_INJ_F) {
                double u[NPT];
                load_chunk<NPT>(cx, right, Cb(c + 1));
                load_chunk<NPT>(cx, u, Ucr(c + 1));
#pragma unroll
                for (int q = 0; q < NPT; ++q) right[q] = __dadd_rn(right[q], u[q]);
                if (last) store_chunk<NPT>(cx, U(tC), right);
            } else if (A.phase == MGRIT_PHASE_F_RES) {
                load_chunk<NPT>(cx, right, Cb(c + 1));
                store_chunk<NPT>(cx, U(tC), right);
            } else {
                if (A.zero_init) {
#pragma unroll
                    for (int q = 0; q < NPT; ++q) right[q] = 0.0;
                    store_chunk<NPT>(cx, U(tC), right);
                } else {
                    load_chunk<NPT>(cx, right, U(tC));
                }
                store_chunk<NPT>(cx, Cb(c + 1), right);
            }
            double ss = 0.0;
            const double *g = Gr(tC);
#pragma unroll
            for (int q = 0; q < NPT; ++q) {
                const int i = cx.base + threadIdx.x + q * NTC;
                const double r = __dsub_rn(__dadd_rn(g ? g[i] : 0.0, v[q]), right[q]);
                v[q] = r;
                ss = __dadd_rn(ss, __dmul_rn(r, r));
            }
            if (A.Gc && A.phase != MGRIT_PHASE_INJ_F) store_chunk<NPT>(cx, A.Gc + (c + 1 - A.c_row0) * (int64_t)n, v);
            if (A.partial) {
                const ArTok tk = ar_send<NPT, 1, false, false>(cx, ss, 0.0, v);
                const double tot = ar_recv<false>(cx, tk).x;
                if (threadIdx.x == 0 && cx.rank == 0) A.partial[c - A.partial0] = tot;
            }
        }
    }
    cluster_sync_all();  // no CTA leaves while peers may still write into it
}

// ------------------------------------------------------ sequential sweep --
template <int P, int NPT, bool NUMBA, bool LOWSYNC, bool GG, int CS>
__global__ void __launch_bounds__(NTC) cl_sweep_kernel(mgrit_level_desc L, double *U, int64_t ldu, const double *G,
                                                       int64_t ldg, int zero_init, int32_t *gmres_iters,
                                                       int32_t *status) {
    const int n = L.n_x;
    ClCtx<CS> cx = make_clctx<CS>(n, L.gmres_max_iters, status);
    cl_init(cx);
    double v[NPT], sv[NPT];
    load_records_chunk<NPT>(cx, L, 0, sv);
    bool have_pub = !zero_init;
    if (zero_init) {
#pragma unroll
        for (int k = 0; k < NPT; ++k) v[k] = 0.0;
        store_chunk<NPT>(cx, U, v);
        zero_row<GG>(cx);
    } else {
        publish_row<GG>(cx, U);
    }
#pragma unroll 1
    for (int64_t t = 0; t < L.n_steps; ++t) {
        const int cnt = cl_apply<P, NPT, NUMBA, LOWSYNC, GG, CS>(L, t, cx, v, sv, have_pub);
        have_pub = true;
        if (t + 1 < L.n_steps) load_records_chunk<NPT>(cx, L, t + 1, sv);
        add_forcing_chunk<NPT>(cx, v, G ? G + (t + 1) * ldg : nullptr);
        store_chunk<NPT>(cx, U + (t + 1) * ldu, v);
        if (gmres_iters && threadIdx.x == 0 && cx.rank == 0) gmres_iters[t] = cnt;
        if (t + 1 < L.n_steps) publish_row<GG>(cx, U + (t + 1) * ldu);
    }
    cluster_sync_all();
}

// ------------------------------------------------------------- launchers --
// Eligible: corrected 1D level whose row splits into CS chunks of 128 x NP
// nodes (NP in {1, 2, 4, 8, 16}) with the Krylov chunk slots in shared
// memory; every row pointer / leading dimension 16-byte aligned (TMA bulk
// copies).
inline bool cl_aligned(const void *p) { return ((uintptr_t)p & 15) == 0; }

template <int CS>
inline int cl_npt(int n) {
    if (n % (CS * NTC)) return 0;
    const int np = n / (CS * NTC);
    return (np == 1 || np == 2 || np == 4 || np == 8 || np == 16) ? np : 0;
}

template <int CS>
inline bool cl_eligible(const mgrit_level_desc *L) {
    // (plain SL levels: the sequential sweep only, see cl_sweep)
    if ((L->kind != MGRIT_KIND_CORRECTED && L->kind != MGRIT_KIND_SL) || L->dim != 1) return false;
    if (!cl_npt<CS>(L->n_x)) return false;
    // (16 nodes per thread leave no registers for the low-sync variant;
    //  those launches run classic MGS, see LaunchCl)
    if (L->gmres_max_iters < 1 || L->gmres_max_iters > kMaxKrylovCl) return false;
    if (cl_smem_bytes<CS>(L->n_x, L->gmres_max_iters) > (size_t)max_smem_optin()) return false;
    return true;
}

template <int P, int CS>
struct LaunchCl {
    static int phase(const mgrit_level_desc *L, const mgrit_phase_args *A, int32_t *status, cudaStream_t st,
                     int max_clusters);
    static int sweep(const mgrit_level_desc *L, double *U, int64_t ldu, const double *G, int64_t ldg,
                     int zero_init, int32_t *gmres_iters, int32_t *status, cudaStream_t st);
    static int resident_clusters(const mgrit_level_desc *L);
};

#ifdef MGRIT_LAUNCHCL_IMPL
template <int CS, typename Fn>
static int cl_dispatch_npt(int n, Fn &&f) {
    switch (cl_npt<CS>(n)) {
        case 1: return f(std::integral_constant<int, 1>{});
        case 2: return f(std::integral_constant<int, 2>{});
        case 4: return f(std::integral_constant<int, 4>{});
        case 8: return f(std::integral_constant<int, 8>{});
        case 16: return f(std::integral_constant<int, 16>{});
        default: set_error("cluster launch: unsupported row length", cudaErrorInvalidValue); return (int)MGRIT_EINVAL;
    }
}

template <int CS, typename K>
static cudaLaunchConfig_t cl_config(K, int grid, size_t smem, cudaStream_t st, cudaLaunchAttribute *attr) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid, 1, 1);
    cfg.blockDim = dim3(NTC, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CS;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cfg;
}

template <int CS, typename Fn>
static int cl_prep(Fn fn, size_t smem) {
    cudaError_t e = cudaFuncSetAttribute((const void *)fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e == cudaSuccess && CS > 8)
        e = cudaFuncSetAttribute((const void *)fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) {
        set_error("cudaFuncSetAttribute(cluster)", e);
        return MGRIT_ECUDA;
    }
    return MGRIT_OK;
}

// GG for the row length that NP nodes per thread imply
template <int CS, int NP>
constexpr bool cl_gg_np() { return cl_gg<CS>(NP * CS * NTC); }

template <int P, int CS>
int LaunchCl<P, CS>::resident_clusters(const mgrit_level_desc *L) {
    const size_t smem = cl_smem_bytes<CS>(L->n_x, L->gmres_max_iters);
    const int r = cl_dispatch_npt<CS>(L->n_x, [&](auto N) {
        constexpr int NP = decltype(N)::value;
        auto fn = cl_phase_kernel<P, NP, false, cl_gg_np<CS, NP>(), CS>;
        if (cl_prep<CS>(fn, smem)) return 0;
        cudaLaunchAttribute attr[1];
        cudaLaunchConfig_t cfg = cl_config<CS>(fn, CS, smem, 0, attr);
        int ncl = 0;
        if (cudaOccupancyMaxActiveClusters(&ncl, (void *)fn, &cfg) != cudaSuccess) {
            cudaGetLastError();
            ncl = 0;
        }
        return ncl;
    });
    return r < 0 ? 0 : r;
}

template <int P, int CS>
int LaunchCl<P, CS>::phase(const mgrit_level_desc *L, const mgrit_phase_args *A, int32_t *status, cudaStream_t st,
                           int max_clusters) {
    const size_t smem = cl_smem_bytes<CS>(L->n_x, L->gmres_max_iters);
    const int rc = cl_dispatch_npt<CS>(L->n_x, [&](auto N) {
        auto launch = [&](auto fn) {
            int r = cl_prep<CS>(fn, smem);
            if (r) return r;
            int64_t ncl = A->c_count < max_clusters ? A->c_count : max_clusters;
            if (ncl < 1) ncl = 1;
            cudaLaunchAttribute attr[1];
            cudaLaunchConfig_t cfg = cl_config<CS>(fn, (int)(ncl * CS), smem, st, attr);
            cudaError_t e = cudaLaunchKernelEx(&cfg, fn, *L, *A, status);
            if (e != cudaSuccess) {
                set_error("cudaLaunchKernelEx(cl_phase)", e);
                return (int)MGRIT_ECUDA;
            }
            return (int)MGRIT_OK;
        };
        constexpr int NP = decltype(N)::value;
        if constexpr (NP <= 8 && !cl_gg_np<CS, NP>()) {
            if (L->gmres_lowsync) return launch(cl_phase_kernel<P, NP, true, false, CS>);
        }
        return launch(cl_phase_kernel<P, NP, false, cl_gg_np<CS, NP>(), CS>);
    });
    if (rc) return rc;
    return check_launch("level_phase(cluster)");
}

template <int P, int CS>
int LaunchCl<P, CS>::sweep(const mgrit_level_desc *L, double *U, int64_t ldu, const double *G, int64_t ldg,
                           int zero_init, int32_t *gmres_iters, int32_t *status, cudaStream_t st) {
    const size_t smem = cl_smem_bytes<CS>(L->n_x, L->gmres_max_iters);
    const bool numba = L->stencil_numba != 0;
    const int rc = cl_dispatch_npt<CS>(L->n_x, [&](auto N) {
        auto launch = [&](auto fn) {
            int r = cl_prep<CS>(fn, smem);
            if (r) return r;
            cudaLaunchAttribute attr[1];
            cudaLaunchConfig_t cfg = cl_config<CS>(fn, CS, smem, st, attr);
            cudaError_t e = cudaLaunchKernelEx(&cfg, fn, *L, U, ldu, G, ldg, zero_init, gmres_iters, status);
            if (e != cudaSuccess) {
                set_error("cudaLaunchKernelEx(cl_sweep)", e);
                return (int)MGRIT_ECUDA;
            }
            return (int)MGRIT_OK;
        };
        constexpr int NP = decltype(N)::value;
        constexpr bool GG = cl_gg_np<CS, NP>();
        if constexpr (NP <= 8 && !GG) {
            if (L->gmres_lowsync) {
                if (numba) return launch(cl_sweep_kernel<P, NP, true, true, false, CS>);
                return launch(cl_sweep_kernel<P, NP, false, true, false, CS>);
            }
        }
        if (numba) return launch(cl_sweep_kernel<P, NP, true, false, GG, CS>);
        return launch(cl_sweep_kernel<P, NP, false, false, GG, CS>);
    });
    if (rc) return rc;
    return check_launch("sequential_sweep(cluster)");
}
#endif  // MGRIT_LAUNCHCL_IMPL

}  // namespace cl
}  // namespace mgrit
