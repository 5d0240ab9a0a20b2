// capi.cu — extern "C" entry points of libmgrit_b200.so (include/mgrit_b200.h)
// that route to the 1D / 2D kernel families, plus small utility kernels.
#include <cstdio>
#include <cstring>

#include "internal.cuh"

namespace mgrit {


static thread_local char g_err[512] = "";

void set_error(const char *what, cudaError_t e) {
    snprintf(g_err, sizeof g_err, "%s: %s (%d)", what, cudaGetErrorString(e), (int)e);
}

int check_launch(const char *what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        set_error(what, e);
        return MGRIT_ECUDA;
    }
    return MGRIT_OK;
}

namespace {

// fixed-order sum: thread t accumulates x[t], x[t+NT], ... then a block tree
constexpr int kSumThreads = 1024;
__global__ void __launch_bounds__(kSumThreads) sum_kernel(const double *x, int64_t n, double *out) {
    __shared__ double red[kSumThreads / 32 + 1];
    double acc = 0.0;
    for (int64_t i = threadIdx.x; i < n; i += kSumThreads) acc = __dadd_rn(acc, x[i]);
    const double tot = block_sum<kSumThreads>(acc, red);
    if (threadIdx.x == 0) out[0] = tot;
}

__global__ void axpy_rows_kernel_impl(double *U, int64_t ldu, int64_t stride, const double *X,
                                 int64_t ldx, int64_t rows, int64_t n) {
    const int64_t total = rows * n;
    for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < total;
         g += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = g / n, i = g - r * n;
        double *u = U + r * stride * ldu + i;
        *u = __dadd_rn(*u, X[r * ldx + i]);
    }
}

}  // namespace

int axpy_rows_impl(double *U, int64_t ldu, int64_t stride, const double *X, int64_t ldx, int64_t rows, int64_t n,
                   cudaStream_t st) {
    if (rows <= 0 || n <= 0) return MGRIT_OK;
    int64_t g = (rows * n + 255) / 256;
    if (g > 148 * 16) g = 148 * 16;
    axpy_rows_kernel_impl<<<(int)g, 256, 0, st>>>(U, ldu, stride, X, ldx, rows, n);
    return check_launch("axpy_rows");
}
}  // namespace mgrit

using namespace mgrit;

extern "C" int mgrit_abi_version(void) { return MGRIT_ABI_VERSION; }

extern "C" const char *mgrit_last_error(void) { return g_err; }

extern "C" int64_t mgrit_gmres_scratch_bytes(const mgrit_level_desc *L, int64_t rows) {
    if (!L) return 0;
    if (L->dim == 2) return scratch2d_bytes(L, rows);
    if (L->kind != MGRIT_KIND_CORRECTED) return 0;
    return rows * (int64_t)(L->gmres_max_iters + 1) * L->n_points * (int64_t)sizeof(double);
}

extern "C" int64_t mgrit_resident_rows(const mgrit_level_desc *L) {
    if (!L) return 0;
    if (L->dim == 2) return capacity2d(L);
    return rows_capacity(L);
}

extern "C" int mgrit_apply_rows(const mgrit_level_desc *L, int64_t B, const int64_t *t_idx,
                                int64_t t_first, int64_t t_stride, const double *U_in,
                                int64_t ld_in, const double *G, int64_t ld_g, const double *U_sub,
                                int64_t ld_sub, double *out, int64_t ld_out, double *row_sumsq,
                                int32_t *gmres_iters, void *scratch, int64_t scratch_bytes,
                                int32_t *status, void *stream) {
    if (!L || B < 0 || (B > 0 && (!U_in || (!out && !row_sumsq))) || !status) return MGRIT_EINVAL;
    RowsArgs a{B, t_idx, t_first, t_stride, U_in, ld_in, G, ld_g, U_sub, ld_sub, out, ld_out,
               row_sumsq, gmres_iters};
    if (L->dim == 1) return apply_rows_1d(L, a, scratch, scratch_bytes, status, (cudaStream_t)stream);
    if (L->dim == 2) return apply_rows_2d(L, a, scratch, scratch_bytes, status, (cudaStream_t)stream);
    snprintf(g_err, sizeof g_err, "apply_rows: dim %d unsupported", L->dim);
    return MGRIT_EINVAL;
}

extern "C" int mgrit_level_phase(const mgrit_level_desc *L, const mgrit_phase_args *A,
                                 void *scratch, int64_t scratch_bytes, int32_t *status,
                                 void *stream) {
    if (!L || !A || !status) return MGRIT_EINVAL;
    if (L->dim == 1) return level_phase_1d(L, A, scratch, scratch_bytes, status, (cudaStream_t)stream);
    if (L->dim == 2) return level_phase_2d(L, A, scratch, scratch_bytes, status, (cudaStream_t)stream);
    snprintf(g_err, sizeof g_err, "level_phase: dim %d unsupported", L->dim);
    return MGRIT_EINVAL;
}

extern "C" int mgrit_sequential_sweep(const mgrit_level_desc *L, double *U, int64_t ldu,
                                      const double *G, int64_t ldg, int32_t zero_init,
                                      int32_t *gmres_iters, void *scratch, int64_t scratch_bytes,
                                      int32_t *status, void *stream) {
    if (!L || !U || !status) return MGRIT_EINVAL;
    if (L->dim == 1)
        return sweep_1d(L, U, ldu, G, ldg, zero_init, gmres_iters, scratch, scratch_bytes, status,
                        (cudaStream_t)stream);
    if (L->dim == 2)
        return sweep_2d(L, U, ldu, G, ldg, zero_init, gmres_iters, scratch, scratch_bytes, status,
                        (cudaStream_t)stream);
    snprintf(g_err, sizeof g_err, "sequential_sweep: dim %d unsupported", L->dim);
    return MGRIT_EINVAL;
}

extern "C" int mgrit_records_separable(int32_t n_x, int64_t n_sets, const double *s_x, const double *s_y,
                                       int32_t *flag, void *stream) {
    return records_separable_2d(n_x, n_sets, s_x, s_y, flag, (cudaStream_t)stream);
}

extern "C" int mgrit_sum(const double *x, int64_t n, double *out, void *stream) {
    if (n < 0 || !out || (n > 0 && !x)) return MGRIT_EINVAL;
    sum_kernel<<<1, kSumThreads, 0, (cudaStream_t)stream>>>(x, n, out);
    return check_launch("sum");
}

extern "C" int mgrit_axpy_rows(double *U, int64_t ldu, int64_t u_stride_rows, const double *X,
                               int64_t ldx, int64_t rows, int64_t n, void *stream) {
    if (rows < 0 || n < 0 || (rows > 0 && (!U || !X))) return MGRIT_EINVAL;
    if (rows == 0 || n == 0) return MGRIT_OK;
    return axpy_rows_impl(U, ldu, u_stride_rows, X, ldx, rows, n, (cudaStream_t)stream);
}
