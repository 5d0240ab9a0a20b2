// setup.cu — device construction of the level hierarchy:
// ERK departure tracing, records from caller coordinates, backtracking,
// phi/sigma accumulation, and the numpy PCG64 initial-iterate stream.
//
// All kernels are elementwise over (set, node) and HBM-bound; they run once
// per hierarchy build, outside the solve's timed region (mgrit.py:345-347).
#include "common.cuh"

namespace mgrit {

namespace {

constexpr int kSetupThreads = 256;

__device__ __forceinline__ double node_coord(int i, double h) {
    // core.py:42-43: x_lo + h * arange(n)
    return __dadd_rn(kXLo, __dmul_rn(h, (double)i));
}

// One backward ERK step of size -dt from time t_start + dt
// (erk_trace_back, semi_lagrangian.py:75-115).
__device__ void erk_trace(int speed, const mgrit_erk_tableau &tb, int dim, double &x,
                          double &y, double t_start, double dt) {
    const double hs = -dt;
    const double t1 = __dadd_rn(t_start, dt);
    double kx[6], ky[6];
    for (int s = 0; s < tb.n_stages; ++s) {
        double xs = x, ys = y;
        for (int j = 0; j < s; ++j) {
            const double a = tb.a[s][j];
            if (a != 0.0) {
                const double coef = __dmul_rn(hs, a);
                xs = __dadd_rn(xs, __dmul_rn(coef, kx[j]));
                if (dim == 2) ys = __dadd_rn(ys, __dmul_rn(coef, ky[j]));
            }
        }
        const double ts = __dadd_rn(t1, __dmul_rn(tb.c[s], hs));
        wave_speed(speed, xs, ys, ts, kx[s], ky[s]);
    }
    double dx = x, dy = y;
    for (int s = 0; s < tb.n_stages; ++s) {
        const double coef = __dmul_rn(hs, tb.b[s]);
        dx = __dadd_rn(dx, __dmul_rn(coef, kx[s]));
        if (dim == 2) dy = __dadd_rn(dy, __dmul_rn(coef, ky[s]));
    }
    x = dx;
    y = dy;
}

__global__ void erk_kernel(int dim, int n_x, int speed, mgrit_erk_tableau tb, int64_t set_first,
                           int64_t n_sets, double dt, int n_sub, double dt_sub, double *s_x,
                           double *s_y, double *disp_x, double *disp_y) {
    const int64_t np = dim == 1 ? (int64_t)n_x : (int64_t)n_x * n_x;
    const int64_t total = np * n_sets;
    const double h = kLen / (double)n_x;
    for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < total;
         g += (int64_t)gridDim.x * blockDim.x) {
        const int64_t set = g / np;
        const int64_t i = g - set * np;
        const double ax = node_coord((int)(dim == 1 ? i : i % n_x), h);
        const double ay = dim == 1 ? 0.0 : node_coord((int)(i / n_x), h);
        double x = ax, y = ay;
        // t_start of the (coarse) step; sub-steps walk backwards in time
        // (mgrit.py:205-207: k = n_sub-1 .. 0, t0 + k*dt_sub)
        const double t0 = __dmul_rn((double)(set_first + set), dt);
        for (int k = n_sub - 1; k >= 0; --k) {
            const double ts = n_sub == 1 ? t0 : __dadd_rn(t0, __dmul_rn((double)k, dt_sub));
            erk_trace(speed, tb, dim, x, y, ts, n_sub == 1 ? dt : dt_sub);
        }
        s_x[g] = scaled_coord(x, h);
        disp_x[g] = __dsub_rn(ax, x);
        if (dim == 2) {
            s_y[g] = scaled_coord(y, h);
            disp_y[g] = __dsub_rn(ay, y);
        }
    }
}

__global__ void coords_kernel(int dim, int n_x, int64_t n_sets, const double *cx,
                              const double *cy, double *s_x, double *s_y, double *disp_x,
                              double *disp_y) {
    const int64_t np = dim == 1 ? (int64_t)n_x : (int64_t)n_x * n_x;
    const int64_t total = np * n_sets;
    const double h = kLen / (double)n_x;
    for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < total;
         g += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = g % np;
        const double ax = node_coord((int)(dim == 1 ? i : i % n_x), h);
        s_x[g] = scaled_coord(cx[g], h);
        disp_x[g] = __dsub_rn(ax, cx[g]);
        if (dim == 2) {
            const double ay = node_coord((int)(i / n_x), h);
            s_y[g] = scaled_coord(cy[g], h);
            disp_y[g] = __dsub_rn(ay, cy[g]);
        }
    }
}

// decompose(grid, coords) from a raw coordinate (backtracking.py:34-35)
__device__ __forceinline__ Dec decompose_coord(double c, int n_x, double h) {
    return decompose_s(scaled_coord(c, h), n_x);
}

__global__ void backtrack_kernel(int dim, int n_x, int m, int64_t n_sets, int child_shared,
                                 const double *cdx, const double *cdy, double *s_x, double *s_y,
                                 double *disp_x, double *disp_y) {
    const int64_t np = dim == 1 ? (int64_t)n_x : (int64_t)n_x * n_x;
    const int64_t total = np * n_sets;
    const double h = kLen / (double)n_x;
    for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < total;
         g += (int64_t)gridDim.x * blockDim.x) {
        const int64_t set = g / np;
        const int64_t i = g - set * np;
        auto child = [&](int k) -> int64_t { return child_shared ? 0 : set * m + k; };
        if (dim == 1) {
            const double ax = node_coord((int)i, h);
            double c = __dsub_rn(ax, cdx[child(m - 1) * np + i]);
            for (int k = m - 2; k >= 0; --k) {
                const double *d = cdx + child(k) * np;
                const Dec e = decompose_coord(c, n_x, h);
                const int west = e.e == 0 ? n_x - 1 : e.e - 1;
                const double upd = __dadd_rn(__dmul_rn(__dsub_rn(1.0, e.eps), d[e.e]),
                                             __dmul_rn(e.eps, d[west]));
                c = __dsub_rn(c, upd);
            }
            s_x[g] = scaled_coord(c, h);
            disp_x[g] = __dsub_rn(ax, c);
        } else {
            const int ix = (int)(i % n_x), iy = (int)(i / n_x);
            const double ax = node_coord(ix, h), ay = node_coord(iy, h);
            double cx = __dsub_rn(ax, cdx[child(m - 1) * np + i]);
            double cy = __dsub_rn(ay, cdy[child(m - 1) * np + i]);
            for (int k = m - 2; k >= 0; --k) {
                const double *dx = cdx + child(k) * np;
                const double *dy = cdy + child(k) * np;
                const Dec ex = decompose_coord(cx, n_x, h);
                const Dec ey = decompose_coord(cy, n_x, h);
                const int64_t west = ex.e == 0 ? n_x - 1 : ex.e - 1;
                const int64_t south = ey.e == 0 ? n_x - 1 : ey.e - 1;
                const int64_t ne = (int64_t)ey.e * n_x + ex.e, nw = (int64_t)ey.e * n_x + west;
                const int64_t se = south * n_x + ex.e, sw = south * n_x + west;
                const double one_e = __dsub_rn(1.0, ex.eps), one_n = __dsub_rn(1.0, ey.eps);
                const double a_ne = __dmul_rn(one_e, one_n);
                const double a_nw = __dmul_rn(ex.eps, one_n);
                const double a_se = __dmul_rn(one_e, ey.eps);
                const double a_sw = __dmul_rn(ex.eps, ey.eps);
                const double ux = __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(a_ne, dx[ne]), __dmul_rn(a_nw, dx[nw])),
                                                      __dmul_rn(a_se, dx[se])),
                                            __dmul_rn(a_sw, dx[sw]));
                const double uy = __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(a_ne, dy[ne]), __dmul_rn(a_nw, dy[nw])),
                                                      __dmul_rn(a_se, dy[se])),
                                            __dmul_rn(a_sw, dy[sw]));
                cx = __dsub_rn(cx, ux);
                cy = __dsub_rn(cy, uy);
            }
            s_x[g] = scaled_coord(cx, h);
            disp_x[g] = __dsub_rn(ax, cx);
            s_y[g] = scaled_coord(cy, h);
            disp_y[g] = __dsub_rn(ay, cy);
        }
    }
}

template <int P>
__global__ void phi_sigma_kernel(int dim, int n_x, int m, int64_t n_sets, int child_shared,
                                 const double *s_x, const double *s_y, const double *cs_x,
                                 const double *cs_y, const double *csig_x, const double *csig_y,
                                 double *sig_x, double *sig_y) {
    const int64_t np = dim == 1 ? (int64_t)n_x : (int64_t)n_x * n_x;
    const int64_t total = np * n_sets;
    for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < total;
         g += (int64_t)gridDim.x * blockDim.x) {
        const int64_t set = g / np;
        const int64_t i = g - set * np;
        for (int ax = 0; ax < dim; ++ax) {
            const double *s = ax == 0 ? s_x : s_y;
            const double *cs = ax == 0 ? cs_x : cs_y;
            const double *csig = ax == 0 ? csig_x : csig_y;
            // phi_vector (coarse_correction.py:92-104): sign = (-1)^(p+1) = +1 for odd p
            double acc = f_poly<P>(decompose_s(s[g], n_x).eps);
            for (int k = 0; k < m; ++k) {
                const int64_t c = child_shared ? 0 : set * m + k;
                acc = __dsub_rn(acc, f_poly<P>(decompose_s(cs[c * np + i], n_x).eps));
            }
            acc = __dmul_rn(1.0, acc);
            // sigma_accumulate (coarse_correction.py:118-127): phi + sum children
            if (csig != nullptr) {
                for (int k = 0; k < m; ++k) {
                    const int64_t c = child_shared ? 0 : set * m + k;
                    acc = __dadd_rn(acc, csig[c * np + i]);
                }
            }
            (ax == 0 ? sig_x : sig_y)[g] = acc;
        }
    }
}

// ---- numpy PCG64 (XSL-RR 128/64) + random() ------------------------------

typedef unsigned __int128 u128;

__device__ __forceinline__ u128 pcg_mult() {
    return ((u128)2549297995355413924ULL << 64) | (u128)4865540595714422341ULL;
}

// state after `delta` LCG steps (standard O(log delta) jump-ahead)
__device__ u128 pcg_advance(u128 state, u128 inc, uint64_t delta) {
    u128 cur_mult = pcg_mult(), cur_plus = inc, acc_mult = 1, acc_plus = 0;
    while (delta > 0) {
        if (delta & 1) {
            acc_mult *= cur_mult;
            acc_plus = acc_plus * cur_mult + cur_plus;
        }
        cur_plus = (cur_mult + 1) * cur_plus;
        cur_mult *= cur_mult;
        delta >>= 1;
    }
    return acc_mult * state + acc_plus;
}

__device__ __forceinline__ double pcg_double(u128 st) {
    const uint64_t hi = (uint64_t)(st >> 64), lo = (uint64_t)st;
    const unsigned rot = (unsigned)(st >> 122);
    const uint64_t x = hi ^ lo;
    const uint64_t out = (x >> rot) | (x << ((64 - rot) & 63));
    return (double)(out >> 11) * (1.0 / 9007199254740992.0);
}

// Warp-interleaved generation: a warp owns kPcgWarpBlock consecutive draws;
// lane l produces draws base + l, base + l + 32, ... by jumping its state 32
// steps at a time (x -> A32 x + C32, the affine map of 32 LCG steps), so
// every store instruction of the warp writes 32 consecutive doubles.
constexpr int64_t kPcgWarpBlock = 32 * 64;

__global__ void pcg64_kernel(uint64_t sh, uint64_t sl, uint64_t ih, uint64_t il, int64_t count,
                             int pm1, double *out) {
    const u128 state0 = ((u128)sh << 64) | sl;
    const u128 inc = ((u128)ih << 64) | il;
    // affine map of 32 steps: advance(x, 32) = a32 * x + c32
    const u128 c32 = pcg_advance(0, inc, 32);
    const u128 a32 = pcg_advance(1, inc, 32) - c32;
    const int lane = threadIdx.x & 31;
    const int64_t warps_total = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int64_t blocks = (count + kPcgWarpBlock - 1) / kPcgWarpBlock;
    for (int64_t wb = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; wb < blocks; wb += warps_total) {
        const int64_t base = wb * kPcgWarpBlock;
        int64_t k = base + lane;
        // state after draw k's step (numpy steps, then outputs)
        u128 st = pcg_advance(state0, inc, (uint64_t)k + 1);
        const int64_t end = base + kPcgWarpBlock < count ? base + kPcgWarpBlock : count;
        for (; k < end; k += 32) {
            double v = pcg_double(st);
            if (pm1) v = __dsub_rn(__dmul_rn(2.0, v), 1.0);
            out[k] = v;
            st = a32 * st + c32;
        }
    }
}

int grid_for(int64_t total) {
    int64_t g = (total + kSetupThreads - 1) / kSetupThreads;
    if (g > 148 * 32) g = 148 * 32;
    if (g < 1) g = 1;
    return (int)g;
}

}  // namespace

}  // namespace mgrit

using namespace mgrit;

extern "C" int mgrit_erk_departures(int32_t dim, int32_t n_x, int32_t speed_id,
                                    const mgrit_erk_tableau *tab, int64_t set_first,
                                    int64_t n_sets, double dt, int32_t n_sub, double dt_sub,
                                    double *s_x, double *s_y, double *disp_x, double *disp_y,
                                    void *stream) {
    if ((dim != 1 && dim != 2) || n_x < 1 || !tab || tab->n_stages < 1 || tab->n_stages > 6 ||
        n_sets < 0 || n_sub < 1 || !s_x || !disp_x || (dim == 2 && (!s_y || !disp_y)))
        return MGRIT_EINVAL;
    if (n_sets == 0) return MGRIT_OK;
    const int64_t np = dim == 1 ? (int64_t)n_x : (int64_t)n_x * n_x;
    erk_kernel<<<grid_for(np * n_sets), kSetupThreads, 0, (cudaStream_t)stream>>>(
        dim, n_x, speed_id, *tab, set_first, n_sets, dt, n_sub, dt_sub, s_x, s_y, disp_x, disp_y);
    return check_launch("erk_departures");
}

extern "C" int mgrit_departures_from_coords(int32_t dim, int32_t n_x, int64_t n_sets,
                                            const double *cx, const double *cy, double *s_x,
                                            double *s_y, double *disp_x, double *disp_y,
                                            void *stream) {
    if ((dim != 1 && dim != 2) || n_x < 1 || n_sets < 0 || !cx || !s_x || !disp_x ||
        (dim == 2 && (!cy || !s_y || !disp_y)))
        return MGRIT_EINVAL;
    if (n_sets == 0) return MGRIT_OK;
    const int64_t np = dim == 1 ? (int64_t)n_x : (int64_t)n_x * n_x;
    coords_kernel<<<grid_for(np * n_sets), kSetupThreads, 0, (cudaStream_t)stream>>>(
        dim, n_x, n_sets, cx, cy, s_x, s_y, disp_x, disp_y);
    return check_launch("departures_from_coords");
}

extern "C" int mgrit_backtrack(int32_t dim, int32_t n_x, int32_t m, int64_t n_sets,
                               int32_t child_shared, const double *child_disp_x,
                               const double *child_disp_y, double *s_x, double *s_y,
                               double *disp_x, double *disp_y, void *stream) {
    if ((dim != 1 && dim != 2) || n_x < 1 || m < 1 || n_sets < 0 || !child_disp_x || !s_x ||
        !disp_x || (dim == 2 && (!child_disp_y || !s_y || !disp_y)))
        return MGRIT_EINVAL;
    if (n_sets == 0) return MGRIT_OK;
    const int64_t np = dim == 1 ? (int64_t)n_x : (int64_t)n_x * n_x;
    backtrack_kernel<<<grid_for(np * n_sets), kSetupThreads, 0, (cudaStream_t)stream>>>(
        dim, n_x, m, n_sets, child_shared, child_disp_x, child_disp_y, s_x, s_y, disp_x, disp_y);
    return check_launch("backtrack");
}

extern "C" int mgrit_phi_sigma(int32_t dim, int32_t n_x, int32_t p, int32_t m, int64_t n_sets,
                               int32_t child_shared, const double *s_x, const double *s_y,
                               const double *child_s_x, const double *child_s_y,
                               const double *child_sig_x, const double *child_sig_y,
                               double *sig_x, double *sig_y, void *stream) {
    if ((dim != 1 && dim != 2) || n_x < 1 || m < 1 || n_sets < 0 || !s_x || !child_s_x ||
        !sig_x || (dim == 2 && (!s_y || !child_s_y || !sig_y)))
        return MGRIT_EINVAL;
    if (n_sets == 0) return MGRIT_OK;
    const int64_t np = dim == 1 ? (int64_t)n_x : (int64_t)n_x * n_x;
    const int grid = grid_for(np * n_sets);
    cudaStream_t st = (cudaStream_t)stream;
    switch (p) {
        case 1: phi_sigma_kernel<1><<<grid, kSetupThreads, 0, st>>>(dim, n_x, m, n_sets, child_shared, s_x, s_y, child_s_x, child_s_y, child_sig_x, child_sig_y, sig_x, sig_y); break;
        case 3: phi_sigma_kernel<3><<<grid, kSetupThreads, 0, st>>>(dim, n_x, m, n_sets, child_shared, s_x, s_y, child_s_x, child_s_y, child_sig_x, child_sig_y, sig_x, sig_y); break;
        case 5: phi_sigma_kernel<5><<<grid, kSetupThreads, 0, st>>>(dim, n_x, m, n_sets, child_shared, s_x, s_y, child_s_x, child_s_y, child_sig_x, child_sig_y, sig_x, sig_y); break;
        default: return MGRIT_EINVAL;
    }
    return check_launch("phi_sigma");
}

extern "C" int mgrit_pcg64_fill(uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi,
                                uint64_t inc_lo, int64_t count, int32_t pm1, double *out,
                                void *stream) {
    if (count < 0 || (count > 0 && !out)) return MGRIT_EINVAL;
    if (count == 0) return MGRIT_OK;
    const int64_t blocks = (count + kPcgWarpBlock - 1) / kPcgWarpBlock;
    pcg64_kernel<<<grid_for(blocks * 32), kSetupThreads, 0, (cudaStream_t)stream>>>(
        state_hi, state_lo, inc_hi, inc_lo, count, pm1, out);
    return check_launch("pcg64_fill");
}
