// ops.cu — operator-level entry points of the reference's public API that sit
// below Level (mgrit_advect/__init__.py:5-16): decompose, interp_weights,
// apply_ImSD, records from a reference DepartureSet's (east, eps), and the
// batched step with per-row GMRES residual histories (gmres_solve's return).
#include <cstdio>

#include "internal.cuh"

namespace mgrit {
namespace {

constexpr int kOpsThreads = 256;

int grid_for(int64_t work) {
    int64_t g = (work + kOpsThreads - 1) / kOpsThreads;
    if (g > 148 * 32) g = 148 * 32;
    return (int)(g < 1 ? 1 : g);
}

// decompose (semi_lagrangian.py:118-137): the scaled coordinate, then east/eps
__global__ void decompose_kernel(int n_x, int64_t count, const double *coords, int64_t *east, double *eps) {
    const double h = kLen / (double)n_x;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
        const Dec d = decompose_s(scaled_coord(coords[i], h), n_x);
        east[i] = d.e;
        eps[i] = d.eps;
    }
}

template <int P>
__global__ void weights_kernel(int64_t count, const double *eps, double *w) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
        double ww[P + 1];
        lagrange_weights<P>(eps[i], ww);
#pragma unroll
        for (int c = 0; c <= P; ++c) w[i * (P + 1) + c] = ww[c];
    }
}

// s from a reference decompose() result.  decompose computed eps = ceil(s) - s,
// which is exact (Sterbenz) wherever ceil(s) <= 2 s, so s = E - eps exactly with
// E the unwrapped east index (east, or n for the wrapped east == 0).  Where the
// subtraction was inexact (s < 1/2, east == 1) s' = 1 - eps is exact and
// re-decomposes to the same (1, eps); east == 0 with eps == 0 (s == 0 or the
// eps >= 1 guard) maps to s' = n, which wraps back to (0, 0).  So every
// record re-derived from s' on the device equals the reference's (east, eps).
__global__ void records_kernel(int n_x, int64_t count, const int64_t *east, const double *eps, double *s) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t e = east[i] == 0 ? n_x : east[i];
        s[i] = __dsub_rn((double)e, eps[i]);
    }
}

__device__ __forceinline__ int wrap_idx(int i, int n) { return i < 0 ? i + n : (i >= n ? i - n : i); }

// (I - diag(sigma) D) v, coarse_correction.py:130-149.  1D: the circulant
// apply_stencil_periodic groups out = c0 v; out += (c+k v(i+k) + c-k v(i-k));
// 2D: dx = (dx + c+k v(x+k)) + c-k v(x-k) along each axis, v - sx dx - sy dy.
template <int P>
__global__ void imsd_kernel(int dim, int n_x, int64_t rows, const double *sig_x, const double *sig_y,
                            const double *v, int64_t ldv, double *out, int64_t ldo) {
    constexpr int RAD = (P + 1) / 2;
    const int64_t n = dim == 1 ? (int64_t)n_x : (int64_t)n_x * n_x;
    const int64_t total = rows * n;
    for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < total; g += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = g / n, i = g - r * n;
        const double *vr = v + r * ldv;
        const double vi = vr[i];
        double res;
        if (dim == 1) {
            double acc = cmul<P>(RAD, vi);
#pragma unroll
            for (int q = 1; q <= RAD; ++q)
                acc = __dadd_rn(acc, __dadd_rn(cmul<P>(RAD + q, vr[wrap_idx((int)i + q, n_x)]),
                                               cmul<P>(RAD - q, vr[wrap_idx((int)i - q, n_x)])));
            res = __dsub_rn(vi, __dmul_rn(sig_x[i], acc));
        } else {
            const int iy = (int)(i / n_x), ix = (int)(i - (int64_t)iy * n_x);
            const double *row = vr + (int64_t)iy * n_x;
            double dx = cmul<P>(RAD, vi), dy = cmul<P>(RAD, vi);
#pragma unroll
            for (int q = 1; q <= RAD; ++q) {
                dx = __dadd_rn(__dadd_rn(dx, cmul<P>(RAD + q, row[wrap_idx(ix + q, n_x)])),
                               cmul<P>(RAD - q, row[wrap_idx(ix - q, n_x)]));
                dy = __dadd_rn(__dadd_rn(dy, cmul<P>(RAD + q, vr[(int64_t)wrap_idx(iy + q, n_x) * n_x + ix])),
                               cmul<P>(RAD - q, vr[(int64_t)wrap_idx(iy - q, n_x) * n_x + ix]));
            }
            res = __dsub_rn(__dsub_rn(vi, __dmul_rn(sig_x[i], dx)), __dmul_rn(sig_y[i], dy));
        }
        out[r * ldo + i] = res;
    }
}

}  // namespace
}  // namespace mgrit

using namespace mgrit;

extern "C" int mgrit_decompose(int32_t n_x, int64_t count, const double *coords, int64_t *east, double *eps,
                               void *stream) {
    if (n_x < 1 || count < 0 || (count > 0 && (!coords || !east || !eps))) return MGRIT_EINVAL;
    if (count == 0) return MGRIT_OK;
    decompose_kernel<<<grid_for(count), kOpsThreads, 0, (cudaStream_t)stream>>>(n_x, count, coords, east, eps);
    return check_launch("decompose");
}

extern "C" int mgrit_interp_weights(int32_t p, int64_t count, const double *eps, double *w, void *stream) {
    if (count < 0 || (count > 0 && (!eps || !w))) return MGRIT_EINVAL;
    if (count == 0) return (p == 1 || p == 3 || p == 5) ? MGRIT_OK : MGRIT_EINVAL;
    const cudaStream_t st = (cudaStream_t)stream;
    switch (p) {
        case 1: weights_kernel<1><<<grid_for(count), kOpsThreads, 0, st>>>(count, eps, w); break;
        case 3: weights_kernel<3><<<grid_for(count), kOpsThreads, 0, st>>>(count, eps, w); break;
        case 5: weights_kernel<5><<<grid_for(count), kOpsThreads, 0, st>>>(count, eps, w); break;
        default: return MGRIT_EINVAL;
    }
    return check_launch("interp_weights");
}

extern "C" int mgrit_records_from_east_eps(int32_t n_x, int64_t count, const int64_t *east, const double *eps,
                                           double *s, void *stream) {
    if (n_x < 1 || count < 0 || (count > 0 && (!east || !eps || !s))) return MGRIT_EINVAL;
    if (count == 0) return MGRIT_OK;
    records_kernel<<<grid_for(count), kOpsThreads, 0, (cudaStream_t)stream>>>(n_x, count, east, eps, s);
    return check_launch("records_from_east_eps");
}

extern "C" int mgrit_apply_imsd(int32_t dim, int32_t n_x, int32_t p, int64_t rows, const double *sig_x,
                                const double *sig_y, const double *v, int64_t ldv, double *out, int64_t ldo,
                                void *stream) {
    if ((dim != 1 && dim != 2) || n_x < 8 || rows < 0) return MGRIT_EINVAL;
    if (rows > 0 && (!sig_x || !v || !out || (dim == 2 && !sig_y))) return MGRIT_EINVAL;
    if (rows == 0) return MGRIT_OK;
    const int64_t n = dim == 1 ? (int64_t)n_x : (int64_t)n_x * n_x;
    const cudaStream_t st = (cudaStream_t)stream;
    const int g = grid_for(rows * n);
    switch (p) {
        case 1: imsd_kernel<1><<<g, kOpsThreads, 0, st>>>(dim, n_x, rows, sig_x, sig_y, v, ldv, out, ldo); break;
        case 3: imsd_kernel<3><<<g, kOpsThreads, 0, st>>>(dim, n_x, rows, sig_x, sig_y, v, ldv, out, ldo); break;
        case 5: imsd_kernel<5><<<g, kOpsThreads, 0, st>>>(dim, n_x, rows, sig_x, sig_y, v, ldv, out, ldo); break;
        default: return MGRIT_EINVAL;
    }
    return check_launch("apply_imsd");
}

extern "C" int mgrit_apply_rows_hist(const mgrit_level_desc *L, int64_t B, const int64_t *t_idx, int64_t t_first,
                                     int64_t t_stride, const double *U_in, int64_t ld_in, double *out,
                                     int64_t ld_out, int32_t *gmres_iters, double *gmres_hist, void *scratch,
                                     int64_t scratch_bytes, int32_t *status, void *stream) {
    if (!L || B < 0 || (B > 0 && (!U_in || !out)) || !status) return MGRIT_EINVAL;
    RowsArgs a{B, t_idx, t_first, t_stride, U_in, ld_in, nullptr, 0, nullptr, 0, out, ld_out, nullptr, gmres_iters};
    a.gmres_hist = gmres_hist;
    if (L->dim == 1) return apply_rows_1d(L, a, scratch, scratch_bytes, status, (cudaStream_t)stream);
    if (L->dim == 2) return apply_rows_2d(L, a, scratch, scratch_bytes, status, (cudaStream_t)stream);
    return MGRIT_EINVAL;
}
