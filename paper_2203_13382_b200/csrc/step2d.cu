// step2d.cu — the 2D hot path (BASELINE configs 4-5: 512^2 and 1024^2 meshes).
//
// A 2D state row (n = n_x^2 = 0.26-1 M fp64, 2-8 MB) does not fit one SM, so
// 2D steps are batched over rows with many CTAs per row:
//  * plain SL: one thread per node, the (p+1)^2 tensor-product gather reads
//    the previous row through L1/L2 (neighbouring nodes share their source
//    window); per-CTA partial sums give deterministic row norms;
//  * forward Euler: SL into scratch, then the explicit correction pass;
//  * corrected (SL + MGS-GMRES on I - diag(sx) Dx - diag(sy) Dy): one
//    cooperative kernel over the batch; each system is split into chunks
//    over the resident CTAs and every MGS inner product is a system-wide,
//    fixed-order reduction (per-warp-block partials, a barrier over the
//    system's CTAs only, ordered sum); systems never wait for each other.
// The fused MGRIT phases are composed on the host from these batched launches
// with strided row pointers (same semantics as the 1D phase_kernel).
#include <cooperative_groups.h>
#include <cuda/atomic>

#include <cstdio>
#include <cstdlib>
#include <type_traits>

#include "internal.cuh"

namespace cg = cooperative_groups;

namespace mgrit {

namespace {

#ifdef MGRIT_PROBE2D
// tools/probe_coop2d.cu: per-CTA globaltimer stamps around every system
// barrier of gmres2d_coop ([cta][2 * barrier]: arrival, release)
constexpr int kProbeBars = 96;
__device__ unsigned long long *g_probe2d = nullptr;
__device__ __forceinline__ unsigned long long probe_now() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#endif

constexpr int kNT2 = 256;       // threads per CTA for 2D kernels
constexpr int kTile2 = 1024;    // nodes per CTA tile (4 per thread)
constexpr int kMaxK2 = 16;

__device__ __forceinline__ int wrapi(int i, int n) { return i < 0 ? i + n : (i >= n ? i - n : i); }

// 2D SL value at node (ix, iy): semi_lagrangian.py:238-253 (x inner, y outer,
// both accumulators start at 0, separately rounded products)
// NX > 0: the mesh width as a compile-time constant (512, 1024: the BASELINE
// meshes), so the row stride of the tap window is an immediate offset
template <int P, int NX = 0>
__device__ __forceinline__ double sl2d_at(const double *u, int nx_rt, double sx, double sy) {
    const int nx = NX > 0 ? NX : nx_rt;
    constexpr int SL = Stencil<P>::L;
    const Dec dx = decompose_s(sx, nx);
    const Dec dy = decompose_s(sy, nx);
    double wx[P + 1], wy[P + 1];
    lagrange_weights<P>(dx.eps, wx);
    lagrange_weights<P>(dy.eps, wy);
    constexpr int R = Stencil<P>::R;
    double out = 0.0;
    if (dx.e >= SL && dx.e + R < nx && dy.e >= SL && dy.e + R < nx) {
        // interior window (almost every node): one base address, the taps
        // are immediate offsets from it and one row stride
        const double *r = u + (int64_t)(dy.e - SL) * nx + (dx.e - SL);
        if constexpr (NX > 0) {
#pragma unroll
            for (int jy = 0; jy <= P; ++jy) {
                double acc = 0.0;
#pragma unroll
                for (int jx = 0; jx <= P; ++jx)
                    acc = __dadd_rn(acc, __dmul_rn(wx[jx], __ldg(r + jy * NX + jx)));  // immediate offsets
                out = __dadd_rn(out, __dmul_rn(wy[jy], acc));
            }
        } else {
#pragma unroll
            for (int jy = 0; jy <= P; ++jy, r += nx) {
                double acc = 0.0;
#pragma unroll
                for (int jx = 0; jx <= P; ++jx) acc = __dadd_rn(acc, __dmul_rn(wx[jx], __ldg(r + jx)));
                out = __dadd_rn(out, __dmul_rn(wy[jy], acc));
            }
        }
        return out;
    }
    int cols[P + 1];
#pragma unroll
    for (int j = 0; j <= P; ++j) cols[j] = wrapi(dx.e - SL + j, nx);
#pragma unroll
    for (int jy = 0; jy <= P; ++jy) {
        const double *r = u + (int64_t)wrapi(dy.e - SL + jy, nx) * nx;
        double acc = 0.0;
#pragma unroll
        for (int jx = 0; jx <= P; ++jx) acc = __dadd_rn(acc, __dmul_rn(wx[jx], __ldg(r + cols[jx])));
        out = __dadd_rn(out, __dmul_rn(wy[jy], acc));
    }
    return out;
}

// (I - diag(sx) Dx - diag(sy) Dy) v at node (ix, iy) (coarse_correction.py:141-149:
// dx = c0 v; dx = dx + c+k v(x+k) + c-k v(x-k); v - sx dx - sy dy)
template <int P>
__device__ __forceinline__ double imsd2d_at(const double *v, int nx, int ix, int iy, double sx, double sy) {
    constexpr int RAD = (P + 1) / 2;
    const double *row = v + (int64_t)iy * nx;
    const double vi = row[ix];
    double dx = cmul<P>(RAD, vi), dy = cmul<P>(RAD, vi);
    if (ix >= RAD && ix + RAD < nx && iy >= RAD && iy + RAD < nx) {
        // interior: immediate offsets from the node's address
        const double *c = row + ix;
#pragma unroll
        for (int q = 1; q <= RAD; ++q) {
            dx = __dadd_rn(__dadd_rn(dx, cmul<P>(RAD + q, c[q])), cmul<P>(RAD - q, c[-q]));
            dy = __dadd_rn(__dadd_rn(dy, cmul<P>(RAD + q, c[(int64_t)q * nx])), cmul<P>(RAD - q, c[-(int64_t)q * nx]));
        }
        return __dsub_rn(__dsub_rn(vi, __dmul_rn(sx, dx)), __dmul_rn(sy, dy));
    }
#pragma unroll
    for (int q = 1; q <= RAD; ++q) {
        dx = __dadd_rn(__dadd_rn(dx, cmul<P>(RAD + q, row[wrapi(ix + q, nx)])), cmul<P>(RAD - q, row[wrapi(ix - q, nx)]));
        dy = __dadd_rn(__dadd_rn(dy, cmul<P>(RAD + q, v[(int64_t)wrapi(iy + q, nx) * nx + ix])),
                       cmul<P>(RAD - q, v[(int64_t)wrapi(iy - q, nx) * nx + ix]));
    }
    return __dsub_rn(__dsub_rn(vi, __dmul_rn(sx, dx)), __dmul_rn(sy, dy));
}

// Same operator applied to b = v / s, each value of b formed exactly as the
// normalisation b_j = w / h would store it (div_rcp, = RN(v / s)); also
// returns b at the node itself.  Lets the GMRES stencil pass read the
// un-normalised Arnoldi vector and write b_kk on the fly (no separate pass).
template <int P, int NX = 0>
__device__ __forceinline__ double imsd2d_scaled(const double *v, int nx_rt, int ix, int iy, double sx, double sy,
                                                double s, double rs, double &bi) {
    const int nx = NX > 0 ? NX : nx_rt;
    constexpr int RAD = (P + 1) / 2;
    const double *row = v + (int64_t)iy * nx;
    auto bq = [&](double x) { return div_rcp(x, s, rs); };
    const double vi = bq(row[ix]);
    bi = vi;
    double dx = cmul<P>(RAD, vi), dy = cmul<P>(RAD, vi);
    if (ix >= RAD && ix + RAD < nx && iy >= RAD && iy + RAD < nx) {
        const double *c = row + ix;
#pragma unroll
        for (int q = 1; q <= RAD; ++q) {
            dx = __dadd_rn(__dadd_rn(dx, cmul<P>(RAD + q, bq(c[q]))), cmul<P>(RAD - q, bq(c[-q])));
            const int64_t qn = NX > 0 ? (int64_t)q * NX : (int64_t)q * nx;
            dy = __dadd_rn(__dadd_rn(dy, cmul<P>(RAD + q, bq(c[qn]))), cmul<P>(RAD - q, bq(c[-qn])));
        }
        return __dsub_rn(__dsub_rn(vi, __dmul_rn(sx, dx)), __dmul_rn(sy, dy));
    }
#pragma unroll
    for (int q = 1; q <= RAD; ++q) {
        dx = __dadd_rn(__dadd_rn(dx, cmul<P>(RAD + q, bq(row[wrapi(ix + q, nx)]))),
                       cmul<P>(RAD - q, bq(row[wrapi(ix - q, nx)])));
        dy = __dadd_rn(__dadd_rn(dy, cmul<P>(RAD + q, bq(v[(int64_t)wrapi(iy + q, nx) * nx + ix]))),
                       cmul<P>(RAD - q, bq(v[(int64_t)wrapi(iy - q, nx) * nx + ix])));
    }
    return __dsub_rn(__dsub_rn(vi, __dmul_rn(sx, dx)), __dmul_rn(sy, dy));
}

struct Rows2D {
    int64_t B;
    const int64_t *t_idx;
    int64_t t_first, t_stride;
    const double *U_in; int64_t ld_in;
    const double *G; int64_t ld_g;
    const double *U_sub; int64_t ld_sub;
    double *out; int64_t ld_out;
    double *partial;  // [B][tiles] row sum-of-squares partials (nullable)
    double *gmres_hist = nullptr;  // [B][K+1] GMRES residual histories (corrected, nullable)
};

__device__ __forceinline__ int64_t row_t(const Rows2D &a, int64_t b) {
    return a.t_idx ? a.t_idx[b] : a.t_first + b * a.t_stride;
}

// plain SL (SLONLY: write S only, no forcing / residual form).
// The step is FP64-issue bound with the tap gathers' L1 latency as the main
// stall, so occupancy and early record loads matter: PREF loads the CTA
// tile's departure records (streaming, read once per phase) before any
// gather, and MINB caps registers for resident CTAs per SM.  Measured on
// B200 per batched F-step (tools/sl2d_variants.py): p = 3 best at 8 CTAs/SM
// (32 regs: cfg4 0.865 -> 0.713 ms), p = 5 at 4 CTAs/SM (64 regs: cfg5
// 5.87 -> 4.99 ms); records loaded lazily were 4-18 % slower.
template <int P>
struct SL2DMinBlocks {
    static constexpr int value = P == 5 ? 4 : 8;
};

// FULL: n is a multiple of the 1024-node tile (every BASELINE 2D mesh), so the
// per-node bounds checks compile away.  Used for p = 5 (cfg5 F-step 4.95 ->
// 4.69 ms); at p = 3 the 32-register build spills more with it and was slower.
template <int P, bool SLONLY, int MINB, bool PREF, bool FULL = false, int NX = 0>
__global__ void __launch_bounds__(kNT2, MINB) sl2d_kernel(mgrit_level_desc L, Rows2D a) {
    __shared__ double red[kNT2 / 32 + 1];
    const int nx = L.n_x;
    const int64_t n = L.n_points;
    const int64_t b = blockIdx.y;
    const int64_t t = row_t(a, b);
    const int64_t set = L.shared ? 0 : t;
    const int64_t tile0 = (int64_t)blockIdx.x * kTile2 + threadIdx.x;
    const double *sx = L.s_x + set * n + tile0, *sy = L.s_y + set * n + tile0;
    const double *u = a.U_in + b * a.ld_in;
    double ss = 0.0;
    constexpr int NK = kTile2 / kNT2;
    double rx[PREF ? NK : 1], ry[PREF ? NK : 1];
    if constexpr (PREF) {
#pragma unroll
        for (int k = 0; k < NK; ++k) {
            const bool in = FULL || tile0 + k * kNT2 < n;
            rx[k] = in ? __ldcs(sx + k * kNT2) : 0.0;
            ry[k] = in ? __ldcs(sy + k * kNT2) : 0.0;
        }
    }
#pragma unroll
    for (int k = 0; k < NK; ++k) {
        const int64_t i = tile0 + k * kNT2;
        if (FULL || i < n) {
            double v = PREF ? sl2d_at<P, NX>(u, nx, rx[k], ry[k])
                            : sl2d_at<P, NX>(u, nx, __ldg(sx + k * kNT2), __ldg(sy + k * kNT2));
            if constexpr (!SLONLY) {
                const double g = a.G ? a.G[b * a.ld_g + i] : 0.0;
                if (a.U_sub) {
                    v = __dsub_rn(__dadd_rn(g, v), a.U_sub[b * a.ld_sub + i]);
                } else {
                    v = __dadd_rn(v, g);
                }
                ss = __dadd_rn(ss, __dmul_rn(v, v));
            }
            if (a.out) a.out[b * a.ld_out + i] = v;
        }
    }
    if constexpr (!SLONLY) {
        if (a.partial) {
            const double tot = block_sum<kNT2>(ss, red);
            if (threadIdx.x == 0) a.partial[b * gridDim.x + blockIdx.x] = tot;
        }
    }
}

// Column-strip SL step: each thread owns NB vertically adjacent nodes of one
// column (a CTA: 256 columns x NB grid rows, warps coalesced along x).
// Where the strip's x-records are bitwise equal (the x-departure does not
// depend on y, e.g. BASELINE's speed (cos^2(pi x)cos(2 pi t) + 0.5, ...))
// and its y-departure rows are consecutive, every node's x-interpolation of
// an absolute source row is the SAME rounded value: the strip computes the
// NB + P row sums once (x-weights once, each tap loaded once) and every node
// combines P + 1 of them with its own y-weights.  The arithmetic of each node
// is exactly the reference's (x inner from 0, y outer from 0, separately
// rounded), so the result is bit-identical; only identical subexpressions
// are shared.  Strips that do not qualify take the per-node path.
// Per node-update at p = 5, NB = 4: ~110 FP64 instructions and ~15 loads
// instead of 185 and 38.
//
// One (row, tile) job per CTA; the job's records are loaded (streaming) before
// anything else.  (A persistent form that prefetched the next job's records
// into shared memory with cp.async measured 1.7x slower on cfg5: 64-register
// spills of the loop state and fewer independent CTAs per SM.)
template <int P, int NB, bool SLONLY, int NX = 0>
__global__ void __launch_bounds__(kNT2, 4) sl2d_strip_kernel(mgrit_level_desc L, Rows2D a, int64_t jobs) {
    __shared__ double red[kNT2 / 32 + 1];
    constexpr int SL = Stencil<P>::L, R = Stencil<P>::R;
    const int nx = NX > 0 ? NX : L.n_x;
    const int64_t n = (int64_t)nx * nx;
    const int tiles_x = nx / kNT2;
    const int64_t tiles = n / ((int64_t)kNT2 * NB);
    const int tid = threadIdx.x;
    {
    const int64_t j = blockIdx.x;
    if (j >= jobs) return;
    const int64_t b = j / tiles, tile = j - b * tiles;
    const int band = (int)(tile / tiles_x);
    const int ix = (int)(tile - (int64_t)band * tiles_x) * kNT2 + tid;
    const int iy0 = band * NB;
    const int64_t set = L.shared ? 0 : row_t(a, b);
    const double *sxp = L.s_x + set * n, *syp = L.s_y + set * n;
    const double *u = a.U_in + b * a.ld_in;
    double sx[NB], sy[NB];
#pragma unroll
    for (int k = 0; k < NB; ++k) {
        const int64_t i = (int64_t)(iy0 + k) * nx + ix;
        sx[k] = __ldcs(sxp + i);
        sy[k] = __ldcs(syp + i);
    }
    bool same = true;
#pragma unroll
    for (int k = 1; k < NB; ++k) same = same && (__double_as_longlong(sx[k]) == __double_as_longlong(sx[0]));
    const Dec dx = decompose_s(sx[0], nx);
    const Dec dy0 = decompose_s(sy[0], nx);
    bool fast = same && dx.e >= SL && dx.e + R < nx;
    double out[NB];
    if (fast) {
        // consecutive y-departure rows (no wrap inside the check: row indices mod n)
#pragma unroll
        for (int k = 1; k < NB; ++k) {
            int want = dy0.e + k;
            if (want >= nx) want -= nx;
            fast = fast && decompose_s(sy[k], nx).e == want;
        }
    }
    if (fast) {
        double wx[P + 1];
        lagrange_weights<P>(dx.eps, wx);
        double acc[NB + P];
#pragma unroll
        for (int r = 0; r < NB + P; ++r) {
            int row = dy0.e - SL + r;
            row = row < 0 ? row + nx : (row >= nx ? row - nx : row);
            const double *src = u + (int64_t)row * nx + (dx.e - SL);
            double s = 0.0;
#pragma unroll
            for (int jx = 0; jx <= P; ++jx) s = __dadd_rn(s, __dmul_rn(wx[jx], __ldg(src + jx)));
            acc[r] = s;
        }
#pragma unroll
        for (int k = 0; k < NB; ++k) {
            const Dec dy = decompose_s(sy[k], nx);
            double wy[P + 1];
            lagrange_weights<P>(dy.eps, wy);
            double o = 0.0;
#pragma unroll
            for (int jy = 0; jy <= P; ++jy) o = __dadd_rn(o, __dmul_rn(wy[jy], acc[k + jy]));
            out[k] = o;
        }
    } else {
#pragma unroll
        for (int k = 0; k < NB; ++k) out[k] = sl2d_at<P, NX>(u, nx, sx[k], sy[k]);
    }
    double ss = 0.0;
#pragma unroll
    for (int k = 0; k < NB; ++k) {
        const int64_t i = (int64_t)(iy0 + k) * nx + ix;
        double v = out[k];
        if constexpr (!SLONLY) {
            const double g = a.G ? a.G[b * a.ld_g + i] : 0.0;
            if (a.U_sub) {
                v = __dsub_rn(__dadd_rn(g, v), a.U_sub[b * a.ld_sub + i]);
            } else {
                v = __dadd_rn(v, g);
            }
            ss = __dadd_rn(ss, __dmul_rn(v, v));
        }
        if (a.out) a.out[b * a.ld_out + i] = v;
    }
    if constexpr (!SLONLY) {
        if (a.partial) {
            const double tot = block_sum<kNT2>(ss, red);
            if (threadIdx.x == 0) a.partial[b * tiles + tile] = tot;
        }
    }
    }
}

// Separable SL step.  When a level's x-records do not depend on the mesh row
// and its y-records do not depend on the column (bitwise; BASELINE's 2D speed
// (cos^2(pi x) cos(2 pi t) + 0.5, sin^2(pi y) cos(2 pi t) + 0.5) traces such
// departures, and mgrit_records_separable() verifies it over every record of
// the level at setup), the tensor-product gather factorises: the
// x-interpolation T[r][ix] = sum_jx wx[ix][jx] u[r][ex(ix) - l + jx] of a
// source row r is the same rounded value for every node of column ix that
// uses row r, and the y-weights of a mesh row are the same in every column.
//
// A CTA owns 256 columns x nb mesh rows, one column per thread.
//   1. The x-record of each column is read from mesh row 0 of the set and the
//      y-record of each row from column 0 (8 B per column / row instead of
//      16 B per node: the step's HBM traffic drops from 32 to 16 B per node).
//   2. The source tile the band touches (nb + p rows plus the drift of the
//      y-departures, 256 + p columns plus the drift of the x-departures) is
//      staged in shared memory with 16-byte cp.async copies, all in flight at
//      once: one DRAM round trip per CTA, four CTAs per SM.
//   3. Each thread slides a register window of p + 1 row sums down its column
//      (every source row is x-interpolated once per column, taps from shared
//      memory); thread k < nb derived mesh row k's y-weights once for the CTA,
//      and every node is the reference's own y-combination of the window.
// Each node's arithmetic is exactly semi_lagrangian.py:238-253 (x inner from
// 0, y outer from 0, separately rounded products), so rows are bit-identical
// to the per-node kernels; only identical subexpressions are shared.  Per
// node-update at p = 5, nb = 16: ~27 FP64 instructions (per-node kernel: 185),
// which takes the step off the FP64-issue bound.
//
// A tile whose source rows or columns do not fit the staged tile (large-CFL
// coarse levels) gathers per node from the same two reference records.
//
// Row norms: partial sums are formed per 256 x kSepSub sub-block, whatever nb
// is, so a row's sum of squares does not depend on the batch size.
constexpr int kSepMaxRows = 32;
constexpr int kSepSub = 8;
constexpr int kSepSlack = 2;   // staged rows beyond nb + p
constexpr int kSepW = 264;     // staged columns (256 + p + drift + alignment), even

__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((unsigned)__cvta_generic_to_shared(smem)), "l"(gmem)
                 : "memory");
}

template <int P, bool SLONLY>
__global__ void __launch_bounds__(kNT2, 4) sl2d_sep_kernel(mgrit_level_desc L, Rows2D a, int nb, int cap, int64_t jobs) {
    extern __shared__ __align__(16) double s_raw[];   // [cap][kSepW] staged source tile
    __shared__ __align__(16) double s_wy[kSepMaxRows][P + 1];
    __shared__ double s_sy[kSepMaxRows];
    __shared__ int s_ey[kSepMaxRows], s_rk[kSepMaxRows];
    __shared__ int s_cmin[kNT2 / 32], s_cmax[kNT2 / 32], s_win[3];
    __shared__ double red[kNT2 / 32 + 1];
    constexpr int SL = Stencil<P>::L;
    const int nx = L.n_x;
    const int64_t n = (int64_t)nx * nx;
    const int tiles_x = nx / kNT2;
    const int64_t tiles = (int64_t)tiles_x * (nx / nb);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t j = blockIdx.x;
    if (j >= jobs) return;
    const int64_t b = j / tiles, tile = j - b * tiles;
    const int band = (int)(tile / tiles_x);
    const int ix = (int)(tile - (int64_t)band * tiles_x) * kNT2 + tid;
    const int iy0 = band * nb;
    const int64_t set = L.shared ? 0 : row_t(a, b);
    const int64_t i0 = (int64_t)iy0 * nx + ix;
    const double *u = a.U_in + b * a.ld_in;

    // column ix's x-record (mesh row 0); mesh row k's y-record (column 0), its
    // east row and weights, and the band's source-row window (warp 0: lane k
    // owns mesh row k): east rows relative to the first one (periodic, nearest
    // image), lowest row and span
    const double sx0 = __ldg(L.s_x + set * n + ix);
    if (warp == 0) {
        const bool act = lane < nb;
        int e = -1;
        if (act) {
            const double s = __ldg(L.s_y + set * n + (int64_t)(iy0 + lane) * nx);
            const Dec d = decompose_s(s, nx);
            double w[P + 1];
            lagrange_weights<P>(d.eps, w);
            s_sy[lane] = s;
            e = (unsigned)d.e < (unsigned)nx ? d.e : -1;
#pragma unroll
            for (int q = 0; q <= P; ++q) s_wy[lane][q] = w[q];
        }
        const int e0 = __shfl_sync(0xffffffffu, e, 0);
        int r = act ? e - e0 : 0;
        if (2 * r < -nx) r += nx;
        if (2 * r > nx) r -= nx;
        const int lo = __reduce_min_sync(0xffffffffu, r), hi = __reduce_max_sync(0xffffffffu, r);
        const bool ok = __all_sync(0xffffffffu, !act || e >= 0);
        if (act) s_rk[lane] = r - lo;   // staged row of the node's first source row
        if (lane == 0) {
            s_win[0] = hi - lo + P + 1;   // span
            s_win[1] = e0 + lo - SL;      // first source row, in (-nx, 2 nx)
            s_win[2] = ok;
        }
    }
    const Dec dx = decompose_s(sx0, nx);
    const bool xok = (unsigned)dx.e < (unsigned)nx;
    // first tap column, as the periodic image nearest to the node's own column
    int c0 = (xok ? dx.e : ix) - SL;
    if (2 * (c0 - ix) > nx) c0 -= nx;
    if (2 * (c0 - ix) < -nx) c0 += nx;
    {
        const int mn = __reduce_min_sync(0xffffffffu, c0), mx = __reduce_max_sync(0xffffffffu, c0);
        if (lane == 0) {
            s_cmin[warp] = mn;
            s_cmax[warp] = mx;
        }
    }
    const bool allx = __syncthreads_and(xok);
    int cmin = s_cmin[0], cmax = s_cmax[0];
#pragma unroll
    for (int w = 1; w < kNT2 / 32; ++w) {
        cmin = min(cmin, s_cmin[w]);
        cmax = max(cmax, s_cmax[w]);
    }
    const int colbase = cmin & ~1;                 // even: 16-byte aligned copies
    const int width = cmax + P + 1 - colbase;      // staged columns
    const int span = s_win[0];
    const bool staged = allx && s_win[2] && span <= cap && width <= kSepW;

    const double *gp = (!SLONLY && a.G) ? a.G + b * a.ld_g + i0 : nullptr;
    const double *up = (!SLONLY && a.U_sub) ? a.U_sub + b * a.ld_sub + i0 : nullptr;
    double *op = a.out ? a.out + b * a.ld_out + i0 : nullptr;
    double *pp = (!SLONLY && a.partial) ? a.partial + b * (n / ((int64_t)kNT2 * kSepSub)) +
                                              (int64_t)(iy0 / kSepSub) * tiles_x + (ix / kNT2)
                                        : nullptr;
    double ss = 0.0;
    // output form of the column's next node (as sl2d_kernel; called for
    // k = 0, 1, .. in order: the row pointers advance) and the sub-block
    // partials.  HG / HS: a forcing row / a row to subtract is present.
    auto emit = [&](auto HG, auto HS, int k, double x) {
        if constexpr (!SLONLY) {
            double g = 0.0;
            if constexpr (decltype(HG)::value) {
                g = *gp;
                gp += nx;
            }
            if constexpr (decltype(HS)::value) {
                x = __dsub_rn(__dadd_rn(g, x), *up);
                up += nx;
            } else {
                x = __dadd_rn(x, g);
            }
            ss = __dadd_rn(ss, __dmul_rn(x, x));
        }
        if (op) {
            *op = x;
            op += nx;
        }
        if constexpr (!SLONLY) {
            if (pp && (k & (kSepSub - 1)) == kSepSub - 1) {
                const double tot = block_sum<kNT2>(ss, red);
                if (tid == 0) *pp = tot;
                pp += tiles_x;
                ss = 0.0;
            }
        }
    };
    // run f(HG, HS) with the output form as compile-time flags
    auto with_form = [&](auto &&f) {
        using T = std::true_type;
        using F = std::false_type;
        if (gp) {
            if (up) f(T{}, T{}); else f(T{}, F{});
        } else {
            if (up) f(F{}, T{}); else f(F{}, F{});
        }
    };
    if (!staged) {   // the band's source window does not fit: per-node gathers
        with_form([&](auto HG, auto HS) {
#pragma unroll 1
            for (int k = 0; k < nb; ++k) emit(HG, HS, k, sl2d_at<P, 0>(u, nx, sx0, s_sy[k]));
        });
        return;
    }

    // stage rows [first, first + span) x columns [colbase, colbase + width) (periodic)
    {
        int first = s_win[1];
        first = first < 0 ? first + nx : (first >= nx ? first - nx : first);
        const int wch = (width + 1) >> 1;   // 16-byte chunks per row
        for (int c = lane; c < wch; c += 32) {
            int col = colbase + 2 * c;
            col = col < 0 ? col + nx : (col >= nx ? col - nx : col);
            const double *src = u + col;
            double *dst = s_raw + 2 * c;
            for (int r = warp; r < span; r += kNT2 / 32) {
                const int row = first + r >= nx ? first + r - nx : first + r;
                cp_async16(dst + r * kSepW, src + (int64_t)row * nx);
            }
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    }
    double wx[P + 1];
    lagrange_weights<P>(dx.eps, wx);
    const double *tcol = s_raw + (c0 - colbase);   // this column's first tap in staged row 0
    auto dot = [&](int r) {
        const double *t = tcol + r * kSepW;
        double acc = 0.0;
#pragma unroll
        for (int q = 0; q <= P; ++q) acc = __dadd_rn(acc, __dmul_rn(wx[q], t[q]));
        return acc;
    };
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncthreads();

    // Window of the row sums of source rows rk .. rk + p of the current node.
    // The slot of source row rk + q rotates with k (slot (k + q) mod (p + 1),
    // static in the unrolled loop), so the usual one-row slide computes one new
    // row sum and moves nothing; any other slide recomputes the window.
    with_form([&](auto HG, auto HS) {
        constexpr int Q = P + 1;
        double W[Q];
        int prev = -2;
        for (int k0 = 0; k0 < nb; k0 += Q) {
#pragma unroll
            for (int jj = 0; jj < Q; ++jj) {
                const int k = k0 + jj;
                if (k < nb) {
                    const int rk = s_rk[k];
                    if (rk - prev == 1) {
                        W[(jj + P) % Q] = dot(rk + P);
                    } else {
#pragma unroll 1
                        for (int q = 0; q < Q; ++q) {   // rare: rebuild the window, oldest row first
#pragma unroll
                            for (int r = 0; r < P; ++r) W[(jj + r) % Q] = W[(jj + r + 1) % Q];
                            W[(jj + P) % Q] = dot(rk + q);
                        }
                    }
                    prev = rk;
                    double o = 0.0;
#pragma unroll
                    for (int q = 0; q < Q; ++q) o = __dadd_rn(o, __dmul_rn(s_wy[k][q], W[(jj + q) % Q]));
                    emit(HG, HS, k, o);
                }
            }
        }
    });
}

// rows per CTA of sl2d_sep_kernel: 16 (a 48 KB table, four CTAs per SM), or 8
// when that leaves SMs without work (MGRIT_SL2D_SEP_ROWS = 8/16/32 overrides, 0 disables
// the kernel)
static int sep_rows(int nx, int64_t B) {
    // read on every call (a getenv is noise next to a launch) so tests can
    // switch the strip height within one process
    const char *e = getenv("MGRIT_SL2D_SEP_ROWS");
    const int env = e ? atoi(e) : -1;
    if (env == 0 || nx % kNT2 != 0) return 0;
    if (env > 0) return (env == 8 || env == 16 || env == 32) && nx % env == 0 ? env : 0;
    for (int nb = 16; nb >= 8; nb >>= 1) {
        if (nx % nb != 0) continue;
        const int64_t jobs = B * (nx / kNT2) * (nx / nb);
        if (jobs >= 2 * 592 || nb == 8) return nb;
    }
    return 0;
}

// strip height of sl2d_strip_kernel (MGRIT_SL2D_STRIP overrides; 0 = the
// per-node kernel).  Measured on B200 (tools/gpu_strip_sweep.sh), cfg5 F-step:
// per-node 4.69 ms, NB = 2 4.11, NB = 4 3.27, NB = 8 3.24 ms (spills; and its
// 64 KB two-stage record buffer exceeds static shared memory): NB = 4.
static int strip_rows() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("MGRIT_SL2D_STRIP");
        v = e ? atoi(e) : 4;
        if (v != 0 && v != 2 && v != 4) v = 4;
    }
    return v;
}

// forward Euler finish: out = (2 v - imsd(v)) [+ G | residual form], v from scratch
template <int P>
__global__ void __launch_bounds__(kNT2) fe2d_kernel(mgrit_level_desc L, Rows2D a, const double *V) {
    __shared__ double red[kNT2 / 32 + 1];
    const int nx = L.n_x;
    const int64_t n = L.n_points;
    const int64_t b = blockIdx.y;
    const int64_t t = row_t(a, b);
    const int64_t set = L.shared ? 0 : t;
    const double *gx = L.sig_x + set * n, *gy = L.sig_y + set * n;
    const double *v = V + b * n;
    double ss = 0.0;
#pragma unroll
    for (int k = 0; k < kTile2 / kNT2; ++k) {
        const int64_t i = (int64_t)blockIdx.x * kTile2 + k * kNT2 + threadIdx.x;
        if (i < n) {
            const int iy = (int)((unsigned)i / (unsigned)nx), ix = (int)i - iy * nx;
            double w = __dsub_rn(__dmul_rn(2.0, v[i]), imsd2d_at<P>(v, nx, ix, iy, __ldg(gx + i), __ldg(gy + i)));
            const double g = a.G ? a.G[b * a.ld_g + i] : 0.0;
            w = a.U_sub ? __dsub_rn(__dadd_rn(g, w), a.U_sub[b * a.ld_sub + i]) : __dadd_rn(w, g);
            ss = __dadd_rn(ss, __dmul_rn(w, w));
            if (a.out) a.out[b * a.ld_out + i] = w;
        }
    }
    if (a.partial) {
        const double tot = block_sum<kNT2>(ss, red);
        if (threadIdx.x == 0) a.partial[b * gridDim.x + blockIdx.x] = tot;
    }
}

// per-row fixed-order sum of the tile partials
__global__ void rowsum_kernel(const double *partial, int tiles, int64_t B, double *row_sumsq) {
    __shared__ double red[kNT2 / 32 + 1];
    for (int64_t b = blockIdx.x; b < B; b += gridDim.x) {
        double acc = 0.0;
        for (int i = threadIdx.x; i < tiles; i += kNT2) acc = __dadd_rn(acc, partial[b * tiles + i]);
        const double tot = block_sum<kNT2>(acc, red);
        if (threadIdx.x == 0) row_sumsq[b] = tot;
    }
}

// ---------------------------------------------------------------------------
// corrected step: cooperative batched MGS-GMRES
//
// Reductions are defined on fixed 256-node "warp blocks" (a warp sums 8
// nodes per lane in a fixed order, then a butterfly), and the system total
// is a fixed-order sum over the warp-block partials.  The result is therefore
// independent of how many CTAs share a system, of the batch size and of the
// rank count in a time-sharded run.

constexpr int kWB = 256;            // nodes per warp block
constexpr int kWBPerLane = kWB / 32;

struct Coop2D {
    mgrit_level_desc L;
    Rows2D a;
    int64_t rows_per_round;   // systems processed concurrently
    int chunks;               // CTAs per system
    int64_t nwb;              // warp blocks per system
    double *basis;            // [rows_per_round][K+1][n]
    double *w;                // [rows_per_round][n] Arnoldi vector (ping)
    double *w2;               // [rows_per_round][n] Arnoldi vector (pong)
    double *part;             // [2][rows_per_round][nwb] reduction partials
    int *flags;               // [rows_per_round][chunks] non-finite rhs
    unsigned int *bar;        // [rows_per_round] per-system barrier counters (zeroed per launch)
    const double *rhs;        // [B][n] right-hand sides S u computed by a batched SL launch (classic kernel), or NULL
    const double *rhs_ss;     // [B] their sums of squares
    int32_t *gmres_iters;
    int32_t *status;
};

struct CoopSmem {
    double cs[kMaxK2], sn[kMaxK2], g[kMaxK2 + 1], y[kMaxK2], H[(kMaxK2 + 1) * kMaxK2];
    double red[kNT2 / 32 + 1];
    int stop;
};

template <int P, int NX = 0>
__global__ void __launch_bounds__(kNT2, 4) gmres2d_coop(Coop2D C) {
    __shared__ CoopSmem S;
    // per warp: a patch + halo of the normalised vector (stencil pass), and the
    // Arnoldi vector w of the warp's first patch (its second patch's w reuses
    // the halo tile, free once that patch's stencil is done)
    constexpr int kTileElems = (32 + (P + 1)) * (kWBPerLane + (P + 1));
    extern __shared__ double s_tile[];   // [kNT2 / 32][kTileElems + kWB] (coop_dyn_smem)
    const mgrit_level_desc &L = C.L;
    const Rows2D &a = C.a;
    const int nx = L.n_x;
    const int64_t n = L.n_points;
    const int K = L.gmres_max_iters;
    const double tol = L.gmres_tol;
    const int slot = blockIdx.x / C.chunks;   // system slot within the round
    const int chunk = blockIdx.x % C.chunks;
    const bool active_cta = slot < C.rows_per_round;
    const int64_t nwb = C.nwb;
    const int64_t wb0 = nwb * chunk / C.chunks, wb1 = nwb * (chunk + 1) / C.chunks;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr int NW = kNT2 / 32;
    int pbuf = 0;

    // Node mapping of a warp block (256 nodes, 8 per lane), fixed per mesh so
    // that every reduction's partials and their order are independent of how
    // many CTAs share a system:
    //  * patch mode (n_x a multiple of 32: every BASELINE mesh): a 32 x 8 patch,
    //    lane = column, k = row.  Patches are numbered along x, so a warp still
    //    reads 256 contiguous bytes per row, and the stencil pass can stage a
    //    patch plus its halo in shared memory (below);
    //  * otherwise 256 consecutive nodes, lane + 32 k.
    const bool patch = (nx % 32) == 0;
    const int pbx = nx / 32;   // patches per patch row
    const bool row_blocks = (nx % kWB) == 0;
    // for every node of this CTA's warp blocks, body(i, ix, iy) -> value; the
    // per-warp-block sum (per lane in k order, then the butterfly) goes to the
    // current partial buffer
    // On-chip w (patch mode, at most two patches per warp): between the stencil
    // pass of an Arnoldi step and its last projection, w = A b_k lives in the
    // shared memory of the warp that owns the nodes (slot 0: its own 256
    // doubles; slot 1: the halo tile), so a projection pass streams only b_j
    // and b_{j+1} from L2 (16 B per node instead of 32).  wp is that node's
    // slot, or nullptr when w stays in global memory.
    const bool onchip = patch && (nwb + C.chunks - 1) / C.chunks <= 2 * NW;
    double *const Ttile = s_tile + warp * (kTileElems + kWB);
    double *const Wown = Ttile + kTileElems;
    auto for_nodes_red = [&](auto &&body) {
        double *pb = C.part + ((int64_t)pbuf * C.rows_per_round + slot) * nwb;
        int sl = 0;
        for (int64_t wb = wb0 + warp; wb < wb1; wb += NW, ++sl) {
            double acc = 0.0;
            if (patch) {
                const int by = (int)(wb / pbx);
                const int ix = ((int)(wb - (int64_t)by * pbx)) * 32 + lane;
                int64_t i = (int64_t)by * kWBPerLane * nx + ix;
                double *wp = onchip ? (sl == 0 ? Wown : Ttile) + lane : nullptr;
#pragma unroll
                for (int k = 0; k < kWBPerLane; ++k, i += nx)
                    acc = __dadd_rn(acc, body(i, ix, by * kWBPerLane + k, wp ? wp + 32 * k : nullptr));
            } else {
                const int64_t base = wb * kWB;
                const int iy0 = row_blocks ? (int)(base / nx) : 0;
                const int ix0 = row_blocks ? (int)(base - (int64_t)iy0 * nx) : 0;
#pragma unroll
                for (int k = 0; k < kWBPerLane; ++k) {
                    const int64_t i = base + lane + 32 * k;
                    if (i < n) {
                        int ix, iy;
                        if (row_blocks) {
                            ix = ix0 + lane + 32 * k;
                            iy = iy0;
                        } else {
                            iy = (int)((unsigned)i / (unsigned)nx);
                            ix = (int)i - iy * nx;
                        }
                        acc = __dadd_rn(acc, body(i, ix, iy, (double *)nullptr));
                    }
                }
            }
            acc = warp_sum(acc);
            if (lane == 0 && active_cta) pb[wb] = acc;
        }
    };
    // Barrier over the `chunks` CTAs of this system slot only (all CTAs are
    // co-resident: cooperative launch).  Monotonic per-slot counter, release
    // on arrival, relaxed polls and one acquire fence at the end (which also
    // invalidates stale L1 lines), so slots never wait for each other: a system that converges
    // early frees HBM bandwidth for the rest instead of idling in lock-step.
    unsigned int gen = 0;
    auto ssync = [&]() {
        __syncthreads();
        if (tid == 0) {
            ++gen;
#ifdef MGRIT_PROBE2D
            if (g_probe2d && gen <= kProbeBars) g_probe2d[((int64_t)blockIdx.x * kProbeBars + gen - 1) * 2] = probe_now();
#endif
            cuda::atomic_ref<unsigned int, cuda::thread_scope_device> ctr(C.bar[slot]);
            ctr.fetch_add(1u, cuda::memory_order_release);
            const unsigned int target = gen * (unsigned int)C.chunks;
            // poll relaxed (every acquire load would invalidate the SM's whole L1,
            // CCTL.IVALL, under the co-resident CTAs that are still gathering taps);
            // one acquire fence once the last arrival is seen
            while (ctr.load(cuda::memory_order_relaxed) < target) {
            }
            cuda::atomic_thread_fence(cuda::memory_order_acquire, cuda::thread_scope_device);
#ifdef MGRIT_PROBE2D
            if (g_probe2d && gen <= kProbeBars) g_probe2d[((int64_t)blockIdx.x * kProbeBars + gen - 1) * 2 + 1] = probe_now();
#endif
        }
        __syncthreads();
    };
    // system barrier, then the fixed-order total of the system's partials
    auto gtotal = [&]() -> double {
        ssync();
        const double *pb = C.part + ((int64_t)pbuf * C.rows_per_round + slot) * nwb;
        double acc = 0.0;
        for (int64_t q = tid; q < nwb; q += kNT2) acc = __dadd_rn(acc, pb[q]);
        const double tot = block_sum<kNT2>(acc, S.red);
        pbuf ^= 1;
        return tot;
    };
    if (!active_cta) return;

    double *basis = C.basis + (int64_t)slot * (K + 1) * n;
    double *const wping = C.w + (int64_t)slot * n, *const wpong = C.w2 + (int64_t)slot * n;
    for (int64_t b = slot; b < a.B; b += C.rows_per_round) {
        const int64_t t = row_t(a, b);
        const int64_t set = L.shared ? 0 : t;
        const double *sx = L.s_x + set * n, *sy = L.s_y + set * n;
        const double *gx = L.sig_x + set * n, *gy = L.sig_y + set * n;
        // ---- SL rhs into w, non-finite flag, beta
        double *src = wping, *dst = wpong;   // Arnoldi vector: read / written by the stencil pass
        double beta;
        int anybad = 0;
        if (C.rhs) {
            // the batch's right-hand sides and their norms come from a batched SL
            // launch of their own (full occupancy, the whole L1 for the taps); the
            // first stencil pass reads the system's row in place, and the row then
            // serves as the second Arnoldi buffer
            src = const_cast<double *>(C.rhs) + b * n;
            dst = wping;
            const double ss = C.rhs_ss[b];
            anybad = !isfinite(ss);     // a non-finite gather value makes the sum non-finite
            beta = sqrt(ss);
        } else {
            int bad = 0;
            const double *u = a.U_in + b * a.ld_in;
            for_nodes_red([&](int64_t i, int ix, int iy, double *wp) {
                const double v = sl2d_at<P, NX>(u, nx, __ldg(sx + i), __ldg(sy + i));
                src[i] = v;
                if (!isfinite(v)) bad = 1;
                return __dmul_rn(v, v);
            });
            bad = __syncthreads_or(bad);
            if (tid == 0) C.flags[(int64_t)slot * C.chunks + chunk] = bad;
            beta = sqrt(gtotal());
            if (tid == 0)
                for (int k = 0; k < C.chunks; ++k) anybad |= C.flags[(int64_t)slot * C.chunks + k];
            anybad = __syncthreads_or(anybad);
        }
        double *hist = (a.gmres_hist && chunk == 0 && tid == 0) ? a.gmres_hist + b * (int64_t)(K + 1) : nullptr;
        if (hist) hist[0] = beta;
        int done = 0;
        const bool skip = anybad || beta == 0.0;
        if (anybad && tid == 0 && chunk == 0) atomicExch(C.status, 1);
        if (tid == 0) S.stop = skip ? 1 : 0;
        double g_k = beta;
        // b_kk = src / scale is never stored by a pass of its own: the stencil
        // pass of iteration kk forms it on the fly from src (every value
        // exactly as the normalisation would store it), writes the node's own
        // b_kk, and writes w = A b_kk into dst.  src was completed before the
        // system barrier inside the gtotal() that produced `scale`.
        double scale = beta, rscale = 1.0 / beta;
        // the stop test is evaluated from the same totals in every CTA of the
        // system, so all of them leave the loop at the same kk
        for (int kk = 0; kk < K; ++kk) {
            __syncthreads();
            if (S.stop) break;
            double *bk = basis + (int64_t)kk * n;
            // b_kk, w = A b_kk ; inner product with b_0
            if (patch) {
                // Each warp forms b = src / scale ONCE for its patch and a halo of
                // the stencil radius (shared memory, (32 + 2r) x (8 + 2r) values
                // for 256 nodes) instead of once per tap (2r(2) + 1 = 13 exact
                // divisions per node at p = 5); the stencil then reads b from
                // shared memory.  Same b values, same stencil arithmetic as
                // imsd2d_scaled: identical w.
                constexpr int RAD = (P + 1) / 2, TW = 32 + 2 * RAD, TH = kWBPerLane + 2 * RAD;
                double *T = Ttile;
                double *pb = C.part + ((int64_t)pbuf * C.rows_per_round + slot) * nwb;
                int sl = 0;
                for (int64_t wb = wb0 + warp; wb < wb1; wb += NW, ++sl) {
                    const int by = (int)(wb / pbx);
                    const int ix0 = ((int)(wb - (int64_t)by * pbx)) * 32, iy0 = by * kWBPerLane;
                    for (int t = lane; t < TW * TH; t += 32) {
                        const int hy = t / TW, hx = t - hy * TW;
                        const int gxx = wrapi(ix0 - RAD + hx, nx), gyy = wrapi(iy0 - RAD + hy, nx);
                        T[t] = div_rcp(src[(int64_t)gyy * nx + gxx], scale, rscale);
                    }
                    __syncwarp();
                    const int ix = ix0 + lane;
                    int64_t i = (int64_t)iy0 * nx + ix;
                    double acc = 0.0;
                    double xk[kWBPerLane];
#pragma unroll
                    for (int k = 0; k < kWBPerLane; ++k, i += nx) {
                        const double *c = T + (k + RAD) * TW + lane + RAD;
                        const double vi = c[0];
                        double dx = cmul<P>(RAD, vi), dy = cmul<P>(RAD, vi);
#pragma unroll
                        for (int q = 1; q <= RAD; ++q) {
                            dx = __dadd_rn(__dadd_rn(dx, cmul<P>(RAD + q, c[q])), cmul<P>(RAD - q, c[-q]));
                            dy = __dadd_rn(__dadd_rn(dy, cmul<P>(RAD + q, c[q * TW])), cmul<P>(RAD - q, c[-q * TW]));
                        }
                        const double x = __dsub_rn(__dsub_rn(vi, __dmul_rn(__ldg(gx + i), dx)), __dmul_rn(__ldg(gy + i), dy));
                        bk[i] = vi;
                        if (onchip)
                            xk[k] = x;
                        else
                            dst[i] = x;
                        acc = __dadd_rn(acc, __dmul_rn(kk == 0 ? vi : basis[i], x));
                    }
                    acc = warp_sum(acc);
                    if (lane == 0) pb[wb] = acc;
                    __syncwarp();   // every lane is done with the tile: it is restaged for the warp's
                                    // next patch, or (second patch) takes that patch's w
                    if (onchip) {
                        double *wp = (sl == 0 ? Wown : T) + lane;
#pragma unroll
                        for (int k = 0; k < kWBPerLane; ++k) wp[32 * k] = xk[k];
                    }
                }
            } else {
                for_nodes_red([&](int64_t i, int ix, int iy, double *wp) {
                    double bi;
                    const double x = imsd2d_scaled<P, NX>(src, nx, ix, iy, __ldg(gx + i), __ldg(gy + i), scale, rscale, bi);
                    bk[i] = bi;
                    dst[i] = x;
                    return __dmul_rn(kk == 0 ? bi : basis[i], x);
                });
            }
            double *const w = dst;
            double hrun = 0.0;
            for (int j = 0; j <= kk; ++j) {
                const double h = gtotal();
                if (tid == 0) {
                    if (j == 0) {
                        hrun = h;
                    } else {
                        const double c = S.cs[j - 1], sn = S.sn[j - 1];
                        const double tmp = __dadd_rn(__dmul_rn(c, hrun), __dmul_rn(sn, h));
                        hrun = __dadd_rn(__dmul_rn(-sn, hrun), __dmul_rn(c, h));
                        S.H[(j - 1) * kMaxK2 + kk] = tmp;
                    }
                }
                // w -= h b_j, fused with the next inner product (b_{j+1} or ||w||^2)
                const double *bj = basis + (int64_t)j * n;
                const double *bn = j < kk ? basis + (int64_t)(j + 1) * n : nullptr;
                if (bn) {
                    for_nodes_red([&](int64_t i, int ix, int iy, double *wp) {
                        const double x = fma(-h, bj[i], wp ? *wp : w[i]);
                        if (wp)
                            *wp = x;
                        else
                            w[i] = x;
                        return __dmul_rn(bn[i], x);
                    });
                } else {
                    for_nodes_red([&](int64_t i, int ix, int iy, double *wp) {
                        // last projection: w goes to memory for the next stencil pass
                        const double x = fma(-h, bj[i], wp ? *wp : w[i]);
                        w[i] = x;
                        return __dmul_rn(x, x);
                    });
                }
            }
            const double nrm = sqrt(gtotal());
            const bool brk = nrm <= __dmul_rn(1e-14, beta);
            // b_{kk+1} = w / nrm is formed by the next stencil pass
            scale = nrm;
            rscale = 1.0 / nrm;
            dst = src;
            src = w;
            if (tid == 0) {
                const double den = hypot(hrun, nrm);
                const double c = __ddiv_rn(hrun, den), sn = __ddiv_rn(nrm, den);
                S.cs[kk] = c;
                S.sn[kk] = sn;
                S.H[kk * kMaxK2 + kk] = den;
                const double gn = __dmul_rn(-sn, g_k);
                S.g[kk] = __dmul_rn(c, g_k);
                S.g[kk + 1] = gn;
                if (hist) hist[kk + 1] = fabs(gn);
                g_k = gn;
                S.stop = brk || (tol >= 0.0 && fabs(gn) <= __dmul_rn(tol, beta));
            }
            done = kk + 1;
        }
        __syncthreads();
        // back substitution (warp 0, column-oriented), x = sum_j b_j y_j, output form
        if (!skip && tid < 32) {
            double acc = lane < done ? S.g[lane] : 0.0;
            for (int j = done - 1; j >= 0; --j) {
                double yj = 0.0;
                if (lane == j) yj = __ddiv_rn(acc, S.H[j * kMaxK2 + j]);
                yj = __shfl_sync(0xffffffffu, yj, j);
                if (lane == j) S.y[j] = yj;
                if (lane < j) acc = __dsub_rn(acc, __dmul_rn(S.H[lane * kMaxK2 + j], yj));
            }
        }
        __syncthreads();
        for_nodes_red([&](int64_t i, int ix, int iy, double *wp) {
            double x = 0.0;
            if (anybad) {
                x = __longlong_as_double(0x7ff8000000000000LL);
            } else if (!skip) {
                for (int j = 0; j < done; ++j) x = fma(basis[(int64_t)j * n + i], S.y[j], x);
            }
            const double g = a.G ? a.G[b * a.ld_g + i] : 0.0;
            x = a.U_sub ? __dsub_rn(__dadd_rn(g, x), a.U_sub[b * a.ld_sub + i]) : __dadd_rn(x, g);
            if (a.out) a.out[b * a.ld_out + i] = x;
            return __dmul_rn(x, x);
        });
        const double tot = gtotal();
        if (tid == 0 && chunk == 0) {
            if (a.partial) a.partial[b] = tot;    // per-row sum of squares
            if (C.gmres_iters) C.gmres_iters[b] = anybad ? -1 : done;
        }
        ssync();  // every chunk is done with this slot's buffers
    }
}

// ---------------------------------------------------------------------------
// Low-synchronisation variant (GmresConfig variant "mgs_lowsync").
//
// The MGS coefficients h_j = <b_j, w - sum_{i<j} h_i b_i> equal, in exact
// arithmetic, c_j - sum_{i<j} h_i G_ji with c_j = <b_j, w> and the Gram
// entries G_ji = <b_j, b_i>.  The stencil pass that forms b_kk and w = A b_kk
// accumulates every c_j (j <= kk) and G_kk,i (i < kk) at once, so an Arnoldi
// step costs two system barriers and two passes (stencil + all inner
// products; w -= sum h_j b_j + ||w||^2) instead of kk + 2 of each.  The
// subtraction w -= h_j b_j runs in the reference's order j = 0..kk.  Results
// equal the classic loop's up to the rounding of the coefficients (GMRES
// iteration counts identical in every parity test, rows within 1e-13).

constexpr int kLsMaxK = 10;                // instantiated Arnoldi depth (K <= 10)
constexpr int kLsVals = 2 * kLsMaxK + 2;   // partial arrays: pass-A bank (2K+1) + bank B

struct LsSmem {
    double cs[kLsMaxK], sn[kLsMaxK], g[kLsMaxK + 1], y[kLsMaxK], H[(kLsMaxK + 1) * kLsMaxK];
    double gram[kLsMaxK * kLsMaxK];        // G_ji = <b_j, b_i>, i < j
    double h[kLsMaxK + 1];
    double red[2 * kLsMaxK + 1][kNT2 / 32];
    int stop;
};

template <int P, int NX = 0>
__global__ void __launch_bounds__(kNT2, 2) gmres2d_coop_ls(Coop2D C) {
    __shared__ LsSmem S;
    const mgrit_level_desc &L = C.L;
    const Rows2D &a = C.a;
    const int nx = L.n_x;
    const int64_t n = L.n_points;
    const int K = L.gmres_max_iters;
    const double tol = L.gmres_tol;
    const int slot = blockIdx.x / C.chunks;
    const int chunk = blockIdx.x % C.chunks;
    const bool active_cta = slot < C.rows_per_round;
    const int64_t nwb = C.nwb;
    const int64_t wb0 = nwb * chunk / C.chunks, wb1 = nwb * (chunk + 1) / C.chunks;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr int NW = kNT2 / 32;
    const bool row_blocks = (nx % kWB) == 0;
    auto part = [&](int v) { return C.part + ((int64_t)v * C.rows_per_round + slot) * nwb; };
    constexpr int kBankB = kLsVals - 1;
    // visit this CTA's nodes; body(i, ix, iy, acc) adds into acc[0..NV) per lane,
    // warp sums land in part(v0 + v)[wb]
    auto for_nodes_nv = [&](auto NVC, int v0, auto &&body) {
        constexpr int NV = decltype(NVC)::value;
        for (int64_t wb = wb0 + warp; wb < wb1; wb += NW) {
            const int64_t base = wb * kWB;
            const int iy0 = row_blocks ? (int)(base / nx) : 0;
            const int ix0 = row_blocks ? (int)(base - (int64_t)iy0 * nx) : 0;
            double acc[NV];
#pragma unroll
            for (int v = 0; v < NV; ++v) acc[v] = 0.0;
#pragma unroll
            for (int k = 0; k < kWBPerLane; ++k) {
                const int64_t i = base + lane + 32 * k;
                if (i < n) {
                    int ix, iy;
                    if (row_blocks) {
                        ix = ix0 + lane + 32 * k;
                        iy = iy0;
                    } else {
                        iy = (int)((unsigned)i / (unsigned)nx);
                        ix = (int)i - iy * nx;
                    }
                    body(i, ix, iy, acc);
                }
            }
#pragma unroll
            for (int v = 0; v < NV; ++v) {
                const double s = warp_sum(acc[v]);
                if (lane == 0 && active_cta) part(v0 + v)[wb] = s;
            }
        }
    };
    unsigned int gen = 0;
    auto ssync = [&]() {
        __syncthreads();
        if (tid == 0) {
            ++gen;
            cuda::atomic_ref<unsigned int, cuda::thread_scope_device> ctr(C.bar[slot]);
            ctr.fetch_add(1u, cuda::memory_order_release);
            const unsigned int target = gen * (unsigned int)C.chunks;
            // poll relaxed (every acquire load would invalidate the SM's whole L1,
            // CCTL.IVALL, under the co-resident CTAs that are still gathering taps);
            // one acquire fence once the last arrival is seen
            while (ctr.load(cuda::memory_order_relaxed) < target) {
            }
            cuda::atomic_thread_fence(cuda::memory_order_acquire, cuda::thread_scope_device);
        }
        __syncthreads();
    };
    // system barrier, then the fixed-order totals of nv partial arrays v0..:
    // per thread a strided sum over the warp blocks, a warp butterfly, then the
    // warp results in warp order (identical in every thread and CTA)
    auto gtotals = [&](int v0, int nv, double *out) {
        ssync();
        for (int v = 0; v < nv; ++v) {
            const double *pb = part(v0 + v);
            double acc = 0.0;
            for (int64_t q = tid; q < nwb; q += kNT2) acc = __dadd_rn(acc, pb[q]);
            acc = warp_sum(acc);
            if (lane == 0) S.red[v][warp] = acc;
        }
        __syncthreads();
        for (int v = 0; v < nv; ++v) {
            double t = 0.0;
#pragma unroll
            for (int w = 0; w < NW; ++w) t = __dadd_rn(t, S.red[v][w]);
            out[v] = t;
        }
        __syncthreads();
    };
    if (!active_cta) return;

    double *basis = C.basis + (int64_t)slot * (K + 1) * n;
    double *const wping = C.w + (int64_t)slot * n, *const wpong = C.w2 + (int64_t)slot * n;
    for (int64_t b = slot; b < a.B; b += C.rows_per_round) {
        const int64_t t = row_t(a, b);
        const int64_t set = L.shared ? 0 : t;
        const double *sx = L.s_x + set * n, *sy = L.s_y + set * n;
        const double *gx = L.sig_x + set * n, *gy = L.sig_y + set * n;
        int bad = 0;
        double *src = wping, *dst = wpong;
        {
            const double *u = a.U_in + b * a.ld_in;
            for_nodes_nv(std::integral_constant<int, 1>{}, kBankB, [&](int64_t i, int, int, double *acc) {
                const double v = sl2d_at<P, NX>(u, nx, __ldg(sx + i), __ldg(sy + i));
                src[i] = v;
                if (!isfinite(v)) bad = 1;
                acc[0] = __dadd_rn(acc[0], __dmul_rn(v, v));
            });
        }
        bad = __syncthreads_or(bad);
        if (tid == 0) C.flags[(int64_t)slot * C.chunks + chunk] = bad;
        double tot[2 * kLsMaxK + 1];
        gtotals(kBankB, 1, tot);
        const double beta = sqrt(tot[0]);
        double *hist = (a.gmres_hist && chunk == 0 && tid == 0) ? a.gmres_hist + b * (int64_t)(K + 1) : nullptr;
        if (hist) hist[0] = beta;
        int anybad = 0;
        if (tid == 0)
            for (int k = 0; k < C.chunks; ++k) anybad |= C.flags[(int64_t)slot * C.chunks + k];
        anybad = __syncthreads_or(anybad);
        int done = 0;
        const bool skip = anybad || beta == 0.0;
        if (anybad && tid == 0 && chunk == 0) atomicExch(C.status, 1);
        if (tid == 0) S.stop = skip ? 1 : 0;
        double g_k = beta;
        double scale = beta, rscale = 1.0 / beta;
        for (int kk = 0; kk < K; ++kk) {
            __syncthreads();
            if (S.stop) break;
            double *bk = basis + (int64_t)kk * n;
            // ---- pass A: b_kk (formed from src / scale), w = A b_kk into dst;
            //      c_j = <b_j, w> (j <= kk) -> arrays 0..kk, G_kk,i = <b_kk, b_i>
            //      (i < kk) -> arrays kk+1..2kk
            auto passA = [&](auto KKC) {
                constexpr int KK = decltype(KKC)::value;
                for_nodes_nv(std::integral_constant<int, 2 * KK + 1>{}, 0,
                             [&](int64_t i, int ix, int iy, double *acc) {
                                 double bi;
                                 const double x = imsd2d_scaled<P, NX>(src, nx, ix, iy, __ldg(gx + i), __ldg(gy + i),
                                                                       scale, rscale, bi);
                                 bk[i] = bi;
                                 dst[i] = x;
#pragma unroll
                                 for (int j = 0; j < KK; ++j) {
                                     const double bj = basis[(int64_t)j * n + i];
                                     acc[j] = fma(bj, x, acc[j]);
                                     acc[KK + 1 + j] = fma(bi, bj, acc[KK + 1 + j]);
                                 }
                                 acc[KK] = fma(bi, x, acc[KK]);
                             });
            };
            switch (kk) {
                case 0: passA(std::integral_constant<int, 0>{}); break;
                case 1: passA(std::integral_constant<int, 1>{}); break;
                case 2: passA(std::integral_constant<int, 2>{}); break;
                case 3: passA(std::integral_constant<int, 3>{}); break;
                case 4: passA(std::integral_constant<int, 4>{}); break;
                case 5: passA(std::integral_constant<int, 5>{}); break;
                case 6: passA(std::integral_constant<int, 6>{}); break;
                case 7: passA(std::integral_constant<int, 7>{}); break;
                case 8: passA(std::integral_constant<int, 8>{}); break;
                default: passA(std::integral_constant<int, 9>{}); break;
            }
            gtotals(0, 2 * kk + 1, tot);
            // MGS coefficients from the inner products and the Gram entries
            // (every thread, identical values)
            double h[kLsMaxK + 1];
            for (int j = 0; j <= kk; ++j) {
                double hj = tot[j];
                for (int i = 0; i < j; ++i) {
                    const double gji = j == kk ? tot[kk + 1 + i] : S.gram[j * kLsMaxK + i];
                    hj = fma(-h[i], gji, hj);
                }
                h[j] = hj;
            }
            __syncthreads();
            if (tid == 0)
                for (int i = 0; i < kk; ++i) S.gram[kk * kLsMaxK + i] = tot[kk + 1 + i];
            // ---- pass B: w -= h_j b_j (j = 0..kk, the reference's order), ||w||^2
            double *const w = dst;
            for_nodes_nv(std::integral_constant<int, 1>{}, kBankB, [&](int64_t i, int, int, double *acc) {
                double x = w[i];
                for (int j = 0; j <= kk; ++j) x = fma(-h[j], basis[(int64_t)j * n + i], x);
                w[i] = x;
                acc[0] = fma(x, x, acc[0]);
            });
            gtotals(kBankB, 1, tot + 2 * kLsMaxK);
            const double nrm = sqrt(tot[2 * kLsMaxK]);
            const bool brk = nrm <= __dmul_rn(1e-14, beta);
            scale = nrm;
            rscale = 1.0 / nrm;
            dst = src;
            src = w;
            if (tid == 0) {
                // previous rotations applied to column kk, then the new one
                double hrun = h[0];
                for (int j = 1; j <= kk; ++j) {
                    const double c = S.cs[j - 1], sn = S.sn[j - 1];
                    const double tmp = __dadd_rn(__dmul_rn(c, hrun), __dmul_rn(sn, h[j]));
                    hrun = __dadd_rn(__dmul_rn(-sn, hrun), __dmul_rn(c, h[j]));
                    S.H[(j - 1) * kLsMaxK + kk] = tmp;
                }
                const double den = hypot(hrun, nrm);
                const double c = __ddiv_rn(hrun, den), sn = __ddiv_rn(nrm, den);
                S.cs[kk] = c;
                S.sn[kk] = sn;
                S.H[kk * kLsMaxK + kk] = den;
                const double gn = __dmul_rn(-sn, g_k);
                S.g[kk] = __dmul_rn(c, g_k);
                S.g[kk + 1] = gn;
                if (hist) hist[kk + 1] = fabs(gn);
                g_k = gn;
                S.stop = brk || (tol >= 0.0 && fabs(gn) <= __dmul_rn(tol, beta));
            }
            done = kk + 1;
        }
        __syncthreads();
        if (!skip && tid < 32) {
            double acc = lane < done ? S.g[lane] : 0.0;
            for (int j = done - 1; j >= 0; --j) {
                double yj = 0.0;
                if (lane == j) yj = __ddiv_rn(acc, S.H[j * kLsMaxK + j]);
                yj = __shfl_sync(0xffffffffu, yj, j);
                if (lane == j) S.y[j] = yj;
                if (lane < j) acc = __dsub_rn(acc, __dmul_rn(S.H[lane * kLsMaxK + j], yj));
            }
        }
        __syncthreads();
        // x = sum_j b_j y_j, output form (bank A: its last readers passed a barrier since)
        for_nodes_nv(std::integral_constant<int, 1>{}, 0, [&](int64_t i, int, int, double *acc) {
            double x = 0.0;
            if (anybad) {
                x = __longlong_as_double(0x7ff8000000000000LL);
            } else if (!skip) {
                for (int j = 0; j < done; ++j) x = fma(basis[(int64_t)j * n + i], S.y[j], x);
            }
            const double g = a.G ? a.G[b * a.ld_g + i] : 0.0;
            x = a.U_sub ? __dsub_rn(__dadd_rn(g, x), a.U_sub[b * a.ld_sub + i]) : __dadd_rn(x, g);
            if (a.out) a.out[b * a.ld_out + i] = x;
            acc[0] = __dadd_rn(acc[0], __dmul_rn(x, x));
        });
        gtotals(0, 1, tot);
        if (tid == 0 && chunk == 0) {
            if (a.partial) a.partial[b] = tot[0];
            if (C.gmres_iters) C.gmres_iters[b] = anybad ? -1 : done;
        }
        ssync();
    }
}

int tiles_for(int64_t n) { return (int)((n + kTile2 - 1) / kTile2); }

int coop_capacity(const void *fn, int smem = 0) {
    int dev = 0, sms = 148, per = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fn, kNT2, smem) != cudaSuccess || per < 1) per = 1;
    return sms * per;
}

template <typename Fn>
int dispatch_p(int p, Fn &&f) {
    switch (p) {
        case 1: return f(std::integral_constant<int, 1>{});
        case 3: return f(std::integral_constant<int, 3>{});
        default: return f(std::integral_constant<int, 5>{});
    }
}

}  // namespace

static int64_t coop_rows_cap(const mgrit_level_desc *L, int64_t grid);

// the cooperative GMRES instantiation a level dispatches to: p = 3 on the
// 512-wide mesh and p = 5 on the 1024-wide mesh use compile-time row strides
static const void *coop_fn(const mgrit_level_desc *L) {
    if (L->gmres_lowsync && L->gmres_max_iters <= kLsMaxK) {
        switch (L->p) {
            case 1: return (const void *)gmres2d_coop_ls<1>;
            case 3: return L->n_x == 512 ? (const void *)gmres2d_coop_ls<3, 512> : (const void *)gmres2d_coop_ls<3>;
            default:
                return L->n_x == 1024 ? (const void *)gmres2d_coop_ls<5, 1024> : (const void *)gmres2d_coop_ls<5>;
        }
    }
    switch (L->p) {
        case 1: return (const void *)gmres2d_coop<1>;
        case 3: return L->n_x == 512 ? (const void *)gmres2d_coop<3, 512> : (const void *)gmres2d_coop<3>;
        default: return L->n_x == 1024 ? (const void *)gmres2d_coop<5, 1024> : (const void *)gmres2d_coop<5>;
    }
}

// dynamic shared memory of the classic cooperative kernel: per warp a patch +
// halo tile and one patch of w (gmres2d_coop); the low-sync kernel uses none
static int coop_dyn_smem(const mgrit_level_desc *L) {
    if (L->gmres_lowsync && L->gmres_max_iters <= kLsMaxK) return 0;
    const int tile = (32 + (L->p + 1)) * (kWBPerLane + (L->p + 1));
    return (kNT2 / 32) * (tile + kWB) * (int)sizeof(double);
}

// opt in to > 48 KB of dynamic shared memory (cheap and idempotent)
static void coop_prepare(const void *fn, int smem) {
    if (smem > 0) cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
}

// systems the corrected 2D kernel keeps in flight: the L2-sized cap (never
// more than the cooperative grid holds), so callers size scratch for exactly
// the rows apply_rows_2d uses
int64_t capacity2d(const mgrit_level_desc *L) {
    if (L->kind != MGRIT_KIND_CORRECTED) return (int64_t)1 << 30;
    coop_prepare(coop_fn(L), coop_dyn_smem(L));
    const int64_t g = coop_capacity(coop_fn(L), coop_dyn_smem(L));
    const int64_t cap = coop_rows_cap(L, g);
    return cap > 0 && cap < g ? cap : g;
}

// Systems solved concurrently by the cooperative kernel: as many as keep
// their working Krylov vectors (~6 of n fp64 each at the tolerance-mode
// iteration counts) inside ~80% of L2, so the MGS passes stream from L2
// rather than HBM (measured on B200: cfg4 64 -> 8 systems 679 -> 618 ms,
// cfg5 32 -> 2 systems 4381 -> 3988 ms per solve).  MGRIT_COOP_ROWS
// overrides (0 = as many as the resident grid allows).
static int64_t coop_rows_cap(const mgrit_level_desc *L, int64_t grid = 0) {
    static int64_t env = -2;
    if (env == -2) {
        const char *e = getenv("MGRIT_COOP_ROWS");
        env = e ? atoll(e) : -1;
    }
    if (env >= 0) return env;
    int dev = 0, l2 = 126 << 20;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev);
    const bool classic = !(L->gmres_lowsync && L->gmres_max_iters <= kLsMaxK);
    // classic loop on a patch-mapped mesh: w lives on chip and the right-hand
    // sides in their own rows, so a system's L2 working set is ~5 vectors; but
    // never so many systems that a warp would own more than two patches
    // (on-chip w needs <= 16 patches per CTA): measured on cfg4, 9 systems in
    // flight 392 ms, 8: 401 ms, 6: 444 ms per solve
    const bool onchip = classic && (L->n_x % 32) == 0;
    const int wv = onchip ? 5 : 6;
    const int vecs = L->gmres_max_iters + 2 < wv ? L->gmres_max_iters + 2 : wv;
    const int64_t per = (int64_t)vecs * L->n_points * 8;
    int64_t r = (int64_t)(0.8 * (double)l2) / (per > 0 ? per : 1);
    if (onchip && grid > 0) {
        const int64_t nwb = (L->n_points + kWB - 1) / kWB;
        const int64_t min_chunks = (nwb + 2 * (kNT2 / 32) - 1) / (2 * (kNT2 / 32));
        const int64_t lim = grid / (min_chunks > 0 ? min_chunks : 1);
        if (lim >= 1 && r > lim) r = lim;
    }
    return r < 1 ? 1 : r;
}

static int64_t coop_row_bytes(const mgrit_level_desc *L) {
    const int64_t n = L->n_points, nwb = (n + kWB - 1) / kWB;
    // basis (K+1) + two Arnoldi vectors, the reduction partials (two banks for
    // the classic loop, 2K+2 arrays for the low-sync one), flags, barrier word
    return 8 * ((int64_t)(L->gmres_max_iters + 3) * n + (int64_t)kLsVals * nwb) + 4 * 4096 + 8;
}

// right-hand sides of a corrected batch: a batched SL launch writes rhs_batch()
// rows S u and their sums of squares ahead of each cooperative launch
// (128 MB of rows: 16 systems of a 1024^2 mesh, 64 of a 512^2 mesh; at most 256)
static int64_t rhs_batch(const mgrit_level_desc *L) {
    const int64_t b = ((int64_t)128 << 20) / (8 * L->n_points);
    return b < 16 ? 16 : (b > 256 ? 256 : b);
}
static int64_t coop_rhs_bytes(const mgrit_level_desc *L) {
    const int64_t n = L->n_points;
    return rhs_batch(L) * (8 * n + 8 + 2 * 8 * tiles_for(n)) + 512;
}

int64_t scratch2d_bytes(const mgrit_level_desc *L, int64_t rows) {
    const int64_t n = L->n_points;
    if (L->kind == MGRIT_KIND_CORRECTED) {
        const int64_t r = rows < 1 ? 1 : rows;
        return r * coop_row_bytes(L) + 4096 + coop_rhs_bytes(L);
    }
    // FE needs the SL rows; all kinds need tile partials for row norms
    const int64_t r = rows < 1 ? 1 : rows;
    // partials: one per 1024-node tile, or per 512-node strip tile (NB = 2)
    return (L->kind == MGRIT_KIND_FORWARD_EULER ? 8 * r * n : 0) + 2 * 8 * r * tiles_for(n) + 256;
}

template <int P, bool SO>
static void launch_strip(int nb, dim3 g, const mgrit_level_desc *L, const Rows2D &s, cudaStream_t st) {
    const int64_t jobs = (int64_t)g.x * g.y;
    auto go = [&](auto NBC) {
        constexpr int NB = decltype(NBC)::value;
        auto run = [&](auto fn) { fn<<<(unsigned)jobs, kNT2, 0, st>>>(*L, s, jobs); };
        if (P == 5 && L->n_x == 1024)
            run(sl2d_strip_kernel<P, NB, SO, (P == 5 ? 1024 : 0)>);
        else if (P == 3 && L->n_x == 512)
            run(sl2d_strip_kernel<P, NB, SO, (P == 3 ? 512 : 0)>);
        else
            run(sl2d_strip_kernel<P, NB, SO, 0>);
    };
    if (nb == 2)
        go(std::integral_constant<int, 2>{});
    else
        go(std::integral_constant<int, 4>{});
}

template <int P, bool SO>
static void launch_sep(int nb, int64_t B, const mgrit_level_desc *L, const Rows2D &s, cudaStream_t st) {
    const int64_t jobs = B * (L->n_x / kNT2) * (L->n_x / nb);
    const int cap = nb + P + kSepSlack;
    const int smem = cap * kSepW * (int)sizeof(double);
    static int optin = 0;   // per instantiation: largest dynamic size opted in so far
    if (smem > optin) {
        cudaFuncSetAttribute(sl2d_sep_kernel<P, SO>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        optin = smem;
    }
    sl2d_sep_kernel<P, SO><<<(unsigned)jobs, kNT2, smem, st>>>(*L, s, nb, cap, jobs);
}

// ---------------------------------------------------------------------------
// separability hint: *flag stays 1 iff, in every record set, s_x does not
// depend on the mesh row and s_y does not depend on the mesh column (bitwise)
__global__ void separable_kernel(int nx, int64_t n_sets, const double *s_x, const double *s_y, int32_t *flag) {
    const int64_t n = (int64_t)nx * nx, total = n_sets * n;
    bool ok = true;
    for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < total; g += (int64_t)gridDim.x * blockDim.x) {
        const int64_t set = g / n, i = g - set * n;
        const int iy = (int)(i / nx), ix = (int)(i - (int64_t)iy * nx);
        const double *bx = s_x + set * n, *by = s_y + set * n;
        ok = ok && __double_as_longlong(bx[i]) == __double_as_longlong(bx[ix]) &&
             __double_as_longlong(by[i]) == __double_as_longlong(by[(int64_t)iy * nx]);
    }
    if (!ok) *flag = 0;
}

__global__ void flag_one_kernel(int32_t *flag) { *flag = 1; }

int records_separable_2d(int32_t n_x, int64_t n_sets, const double *s_x, const double *s_y, int32_t *flag,
                         cudaStream_t st) {
    if (n_x < 8 || n_sets < 1 || !s_x || !s_y || !flag) return MGRIT_EINVAL;
    flag_one_kernel<<<1, 1, 0, st>>>(flag);
    const int64_t total = n_sets * (int64_t)n_x * n_x;
    const int64_t blocks = (total + kNT2 - 1) / kNT2;
    separable_kernel<<<(unsigned)(blocks < 148 * 16 ? blocks : 148 * 16), kNT2, 0, st>>>(n_x, n_sets, s_x, s_y, flag);
    return check_launch("separable_kernel");
}

static int validate2d(const mgrit_level_desc *L) {
    if (!L || L->dim != 2 || L->n_x < 8 || !L->s_x || !L->s_y) return MGRIT_EINVAL;
    if (L->p != 1 && L->p != 3 && L->p != 5) return MGRIT_EINVAL;
    if (L->kind < 0 || L->kind > 2) return MGRIT_EINVAL;
    if (L->kind != MGRIT_KIND_SL && (!L->sig_x || !L->sig_y)) return MGRIT_EINVAL;
    if (L->kind == MGRIT_KIND_CORRECTED && (L->gmres_max_iters < 1 || L->gmres_max_iters > kMaxK2))
        return MGRIT_EINVAL;
    return MGRIT_OK;
}

int apply_rows_2d(const mgrit_level_desc *L, const RowsArgs &r, void *scratch, int64_t scratch_bytes,
                  int32_t *status, cudaStream_t st) {
    int rc = validate2d(L);
    if (rc) return rc;
    if (r.B <= 0) return MGRIT_OK;
    const int64_t n = L->n_points;
    const int tiles = tiles_for(n);
    Rows2D a{r.B, r.t_idx, r.t_first, r.t_stride, r.U_in, r.ld_in, r.G, r.ld_g, r.U_sub, r.ld_sub,
             r.out, r.ld_out, nullptr};
    char *scr = (char *)scratch;
    if (L->kind == MGRIT_KIND_CORRECTED) {
        {
            const void *fn = coop_fn(L);
            const int smem = coop_dyn_smem(L);
            coop_prepare(fn, smem);
            const int G = coop_capacity(fn, smem);
            // the classic loop takes its right-hand sides from a batched SL launch when
            // the scratch holds the batch region (scratch2d_bytes sizes it)
            static int rhs_on = -1;
            if (rhs_on < 0) {
                const char *e = getenv("MGRIT_COOP_RHS_LAUNCH");
                rhs_on = e ? atoi(e) != 0 : 1;
            }
            const bool classic = !(L->gmres_lowsync && L->gmres_max_iters <= kLsMaxK);
            const int64_t per_row = coop_row_bytes(L);
            const int64_t rhs_bytes = coop_rhs_bytes(L);
            const bool rhs_launch = rhs_on && classic && scratch_bytes >= per_row + 4096 + rhs_bytes;
            const int64_t coop_bytes = rhs_launch ? scratch_bytes - rhs_bytes : scratch_bytes;
            int64_t rows = r.B < G ? r.B : G;
            const int64_t cap = coop_rows_cap(L, G);
            if (cap > 0 && rows > cap) rows = cap;
            if (coop_bytes - 4096 < per_row) return (int)MGRIT_EINVAL;
            if (rows > (coop_bytes - 4096) / per_row) rows = (coop_bytes - 4096) / per_row;
            int chunks = (int)(G / rows);
            if (chunks < 1) chunks = 1;
            while ((int64_t)chunks * rows > 4096) --chunks;
            const int64_t nwb = (n + kWB - 1) / kWB;
            Coop2D C;
            C.L = *L;
            C.rows_per_round = rows;
            C.chunks = chunks;
            C.nwb = nwb;
            C.basis = (double *)scr;
            C.w = C.basis + rows * (int64_t)(L->gmres_max_iters + 1) * n;
            C.w2 = C.w + rows * n;
            C.part = C.w2 + rows * n;
            C.flags = (int *)(C.part + (int64_t)kLsVals * rows * nwb);
            C.bar = (unsigned int *)(C.flags + rows * chunks);
            C.status = status;
            C.rhs = nullptr;
            C.rhs_ss = nullptr;
            double *rhs = nullptr, *rhs_ss = nullptr;
            char *rhs_scr = nullptr;
            if (rhs_launch) {
                rhs = (double *)(((uintptr_t)(scr + coop_bytes) + 255) & ~(uintptr_t)255);
                rhs_ss = rhs + rhs_batch(L) * n;
                rhs_scr = (char *)(rhs_ss + rhs_batch(L));
            }
            const int64_t step = rhs_launch ? rhs_batch(L) : r.B;
            const int K1 = L->gmres_max_iters + 1;
            for (int64_t off = 0; off < r.B; off += step) {
                const int64_t cnt = r.B - off < step ? r.B - off : step;
                const int64_t *tix = r.t_idx ? r.t_idx + off : nullptr;
                const int64_t tf = r.t_first + off * r.t_stride;
                if (rhs_launch) {
                    mgrit_level_desc Ls = *L;
                    Ls.kind = MGRIT_KIND_SL;
                    RowsArgs rr{cnt, tix, tf, r.t_stride, r.U_in + off * r.ld_in, r.ld_in, nullptr, 0, nullptr, 0,
                                rhs, n, rhs_ss, nullptr};
                    const int rc2 = apply_rows_2d(&Ls, rr, rhs_scr, 2 * 8 * cnt * tiles_for(n) + 256, status, st);
                    if (rc2) return rc2;
                    C.rhs = rhs;
                    C.rhs_ss = rhs_ss;
                }
                C.a = Rows2D{cnt, tix, tf, r.t_stride, r.U_in + off * r.ld_in, r.ld_in,
                             r.G ? r.G + off * r.ld_g : nullptr, r.ld_g, r.U_sub ? r.U_sub + off * r.ld_sub : nullptr,
                             r.ld_sub, r.out ? r.out + off * r.ld_out : nullptr, r.ld_out,
                             r.row_sumsq ? r.row_sumsq + off : nullptr};
                C.a.gmres_hist = r.gmres_hist ? r.gmres_hist + off * K1 : nullptr;
                C.gmres_iters = r.gmres_iters ? r.gmres_iters + off : nullptr;
                if (cudaMemsetAsync(C.bar, 0, rows * sizeof(unsigned int), st) != cudaSuccess) {
                    set_error("cudaMemsetAsync", cudaGetLastError());
                    return (int)MGRIT_ECUDA;
                }
                void *args[] = {&C};
                const int grid = (int)(rows * chunks);
                cudaError_t e = cudaLaunchCooperativeKernel(fn, grid, kNT2, args, smem, st);
                if (e != cudaSuccess) {
                    set_error("gmres2d_coop", e);
                    return (int)MGRIT_ECUDA;
                }
            }
            return check_launch("gmres2d_coop");
        }
    }
    double *partial = nullptr;
    double *V = nullptr;
    if (L->kind == MGRIT_KIND_FORWARD_EULER) {
        V = (double *)scr;
        scr += 8 * r.B * n;
    }
    if (r.row_sumsq) partial = (double *)scr;
    // column-strip form on meshes whose width is a multiple of the 256-column
    // CTA (every BASELINE 2D mesh); the per-node kernel elsewhere
    const int nb = strip_rows();
    const bool strip = nb > 0 && L->n_x % kNT2 == 0 && L->n_x % nb == 0;
    // separable records (hinted by the level): the sliding-window kernel
    // (16-byte cp.async staging needs 16-byte aligned input rows)
    const bool al16 = ((uintptr_t)r.U_in & 15) == 0 && (r.ld_in & 1) == 0;
    const int sepnb = L->sl2d_separable && al16 ? sep_rows(L->n_x, r.B) : 0;
    const int64_t ptiles = sepnb ? n / ((int64_t)kNT2 * kSepSub) : strip ? n / ((int64_t)kNT2 * nb) : tiles;
    const int64_t need = (V ? 8 * r.B * n : 0) + (partial ? 8 * r.B * ptiles : 0);
    if (need > scratch_bytes) return MGRIT_EINVAL;
    const dim3 grid((unsigned)tiles, (unsigned)r.B);
    const dim3 sgrid((unsigned)ptiles, (unsigned)r.B);
    return dispatch_p(L->p, [&](auto PP) {
        constexpr int P = decltype(PP)::value;
        if (L->kind == MGRIT_KIND_FORWARD_EULER) {
            Rows2D s = a;
            s.out = V;
            s.ld_out = n;
            if (sepnb)
                launch_sep<P, true>(sepnb, r.B, L, s, st);
            else if (strip)
                launch_strip<P, true>(nb, sgrid, L, s, st);
            else if (P == 5 && n % kTile2 == 0)
                sl2d_kernel<P, true, SL2DMinBlocks<P>::value, true, P == 5><<<grid, kNT2, 0, st>>>(*L, s);
            else
                sl2d_kernel<P, true, SL2DMinBlocks<P>::value, true><<<grid, kNT2, 0, st>>>(*L, s);
            Rows2D f = a;
            f.partial = partial;
            fe2d_kernel<P><<<grid, kNT2, 0, st>>>(*L, f, V);
            if (partial) rowsum_kernel<<<(unsigned)(r.B < 4096 ? r.B : 4096), kNT2, 0, st>>>(partial, tiles, r.B, r.row_sumsq);
            return check_launch("apply_rows_2d");
        }
        Rows2D s = a;
        s.partial = partial;
        if (sepnb) {
            launch_sep<P, false>(sepnb, r.B, L, s, st);
        } else if (strip) {
            launch_strip<P, false>(nb, sgrid, L, s, st);
        } else if (P == 3 && L->n_x == 512) {
            // p = 3 on the 512-wide mesh (cfg4): the tap rows are immediate
            // offsets from one base pointer (0.676 -> 0.618 ms per F-step);
            // at p = 5 the same form measured slower (4.69 -> 4.91 ms)
            sl2d_kernel<P, false, SL2DMinBlocks<P>::value, true, false, 512><<<grid, kNT2, 0, st>>>(*L, s);
        } else if (P == 5 && n % kTile2 == 0) {
            sl2d_kernel<P, false, SL2DMinBlocks<P>::value, true, P == 5><<<grid, kNT2, 0, st>>>(*L, s);
        } else {
            sl2d_kernel<P, false, SL2DMinBlocks<P>::value, true><<<grid, kNT2, 0, st>>>(*L, s);
        }
        if (partial)
            rowsum_kernel<<<(unsigned)(r.B < 4096 ? r.B : 4096), kNT2, 0, st>>>(partial, (int)ptiles, r.B, r.row_sumsq);
        return check_launch("apply_rows_2d");
    });
}

// ---------------------------------------------------------------------------
// fused phases for 2D, composed from batched row launches

static int copy_rows(double *dst, int64_t ld_dst, const double *src, int64_t ld_src, int64_t rows, int64_t n,
                     cudaStream_t st) {
    if (rows <= 0) return MGRIT_OK;
    cudaError_t e = cudaMemcpy2DAsync(dst, ld_dst * 8, src, ld_src * 8, n * 8, rows, cudaMemcpyDeviceToDevice, st);
    if (e != cudaSuccess) {
        set_error("cudaMemcpy2DAsync", e);
        return MGRIT_ECUDA;
    }
    return MGRIT_OK;
}

static int zero_rows(double *dst, int64_t ld, int64_t rows, int64_t n, cudaStream_t st) {
    if (rows <= 0) return MGRIT_OK;
    cudaError_t e = cudaMemset2DAsync(dst, ld * 8, 0, n * 8, rows, st);
    if (e != cudaSuccess) {
        set_error("cudaMemset2DAsync", e);
        return MGRIT_ECUDA;
    }
    return MGRIT_OK;
}

int axpy_rows_impl(double *U, int64_t ldu, int64_t stride, const double *X, int64_t ldx, int64_t rows,
                   int64_t n, cudaStream_t st);

int level_phase_2d(const mgrit_level_desc *L, const mgrit_phase_args *A, void *scratch, int64_t scratch_bytes,
                   int32_t *status, cudaStream_t st) {
    int rc = validate2d(L);
    if (rc) return rc;
    if (!A || A->m < 1 || !A->U || !A->Cbuf || A->c_count < 0 || A->n_intervals < 1) return MGRIT_EINVAL;
    if ((int64_t)A->n_intervals * A->m != L->n_steps) return MGRIT_EINVAL;
    if (A->c_count == 0) return MGRIT_OK;
    const int64_t n = L->n_points, m = A->m, cb = A->c_begin, cnt = A->c_count;
    const int64_t ldm = m * A->ldu;
    auto Urow = [&](int64_t t) { return A->U + (t - A->u_row0) * A->ldu; };
    auto Grow = [&](int64_t t) -> const double * { return A->G ? A->G + (t - A->g_row0) * A->ldg : nullptr; };
    auto Crow = [&](int64_t c) { return A->Cbuf + (c - A->c_row0) * n; };
    auto Ucrow = [&](int64_t c) { return A->Uc + (c - A->c_row0) * n; };
    const int64_t ldgm = m * A->ldg;
    auto steps = [&](int64_t k, double *out, int64_t ld_out, const double *Usub, int64_t ld_sub, double *rss) {
        // rows t = c*m + k - 1 -> out; forcing G[c*m + k]
        RowsArgs r{cnt, nullptr, cb * m + k - 1, m, Urow(cb * m + k - 1), ldm, Grow(cb * m + k), ldgm,
                   Usub, ld_sub, out, ld_out, rss, nullptr};
        return apply_rows_2d(L, r, scratch, scratch_bytes, status, st);
    };
    const int phase = A->phase;
    // ---- left states
    if (phase == MGRIT_PHASE_FC || phase == MGRIT_PHASE_FONLY_RES) {
        if (A->zero_init && (rc = zero_rows(Urow(cb * m), ldm, cnt, n, st))) return rc;
    } else if (phase == MGRIT_PHASE_F_RES) {
        if (A->zero_init && cb == 0 && (rc = zero_rows(Urow(0), A->ldu, 1, n, st))) return rc;
        const int64_t c_lo = cb > 0 ? cb : 1;
        if ((rc = copy_rows(Urow(c_lo * m), ldm, Crow(c_lo), n, cb + cnt - c_lo, n, st))) return rc;
    } else if (phase == MGRIT_PHASE_INJ_F) {
        // U[c m] += Uc[c] for c in [cb, cb+cnt] (the right edge too, on this
        // rank's copy, so the C-point residual of its last interval is current)
        if ((rc = axpy_rows_impl(Urow(cb * m), A->ldu, m, Ucrow(cb), n, cnt + 1, n, st))) return rc;
    }
    // ---- F-relaxation (skipped by an FC phase whose F-points are known to
    // hold it already: the steps would rewrite identical rows)
    if (!(phase == MGRIT_PHASE_FC && A->f_relaxed && !A->zero_init))
        for (int64_t k = 1; k < m; ++k) {
            if (k == 1 && A->zero_init && (phase == MGRIT_PHASE_FC || phase == MGRIT_PHASE_FONLY_RES) &&
                L->kind != MGRIT_KIND_FORWARD_EULER) {
                // the left C rows are zero: Phi 0 = +0.0 (an SL gather of zeros; GMRES returns
                // x = 0 at beta = 0, _kernels.py:123-128), so the step's row is 0.0 + g
                if ((rc = zero_rows(Urow(cb * m + 1), ldm, cnt, n, st))) return rc;
                if (A->G && (rc = axpy_rows_impl(Urow(cb * m + 1), A->ldu, m, Grow(cb * m + 1), ldgm, cnt, n, st)))
                    return rc;
                continue;
            }
            if ((rc = steps(k, Urow(cb * m + k), ldm, nullptr, 0, nullptr))) return rc;
        }
    // ---- tails
    if (phase == MGRIT_PHASE_FC) {
        RowsArgs r{cnt, nullptr, cb * m + m - 1, m, Urow(cb * m + m - 1), ldm, Grow(cb * m + m), ldgm,
                   nullptr, 0, Crow(cb + 1), n, nullptr, nullptr};
        return apply_rows_2d(L, r, scratch, scratch_bytes, status, st);
    }
    if (phase == MGRIT_PHASE_F_RES) {
        if ((rc = copy_rows(Urow((cb + 1) * m), ldm, Crow(cb + 1), n, cnt, n, st))) return rc;
    } else if (phase == MGRIT_PHASE_FONLY_RES) {
        if (A->zero_init && (rc = zero_rows(Urow((cb + 1) * m), ldm, cnt, n, st))) return rc;
        if ((rc = copy_rows(Crow(cb + 1), n, Urow((cb + 1) * m), ldm, cnt, n, st))) return rc;
    } else if (phase == MGRIT_PHASE_INJ_F && !A->partial) {
        return MGRIT_OK;
    }
    double *out = (phase == MGRIT_PHASE_INJ_F || !A->Gc) ? nullptr : A->Gc + (cb + 1 - A->c_row0) * n;
    double *rss = A->partial ? A->partial + (cb - A->partial0) : nullptr;
    if (!out && !rss) return MGRIT_OK;
    return steps(m, out, n, Urow((cb + 1) * m), ldm, rss);
}

int sweep_2d(const mgrit_level_desc *L, double *U, int64_t ldu, const double *G, int64_t ldg, int zero_init,
             int32_t *gmres_iters, void *scratch, int64_t scratch_bytes, int32_t *status, cudaStream_t st) {
    int rc = validate2d(L);
    if (rc) return rc;
    const int64_t n = L->n_points;
    if (zero_init && (rc = zero_rows(U, ldu, 1, n, st))) return rc;
    for (int64_t t = 0; t < L->n_steps; ++t) {
        RowsArgs r{1, nullptr, t, 1, U + t * ldu, ldu, G ? G + (t + 1) * ldg : nullptr, ldg, nullptr, 0,
                   U + (t + 1) * ldu, ldu, nullptr, gmres_iters ? gmres_iters + t : nullptr};
        if ((rc = apply_rows_2d(L, r, scratch, scratch_bytes, status, st))) return rc;
    }
    return MGRIT_OK;
}

}  // namespace mgrit
