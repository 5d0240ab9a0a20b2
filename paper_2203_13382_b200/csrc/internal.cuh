// internal.cuh — declarations shared between the kernel families and capi.cu.
#pragma once
#include "common.cuh"

namespace mgrit {

struct RowsArgs {
    int64_t B;
    const int64_t *t_idx;
    int64_t t_first, t_stride;
    const double *U_in; int64_t ld_in;
    const double *G; int64_t ld_g;
    const double *U_sub; int64_t ld_sub;
    double *out; int64_t ld_out;
    double *row_sumsq;
    int32_t *gmres_iters;
    double *gmres_hist = nullptr;   // [B][K+1] GMRES residual histories (corrected rows)
};

int apply_rows_1d(const mgrit_level_desc *L, const RowsArgs &a, void *scratch,
                  int64_t scratch_bytes, int32_t *status, cudaStream_t st);
int level_phase_1d(const mgrit_level_desc *L, const mgrit_phase_args *A, void *scratch,
                   int64_t scratch_bytes, int32_t *status, cudaStream_t st);
int sweep_1d(const mgrit_level_desc *L, double *U, int64_t ldu, const double *G, int64_t ldg,
             int zero_init, int32_t *gmres_iters, void *scratch, int64_t scratch_bytes,
             int32_t *status, cudaStream_t st);
int64_t rows_capacity(const mgrit_level_desc *L);      // incl. the two-CTAs-per-SM phase form
int64_t rows_capacity_one(const mgrit_level_desc *L);  // one-CTA-per-SM forms only
// cluster-split corrected 1D kernels; return -1 when not applicable
int cl_level_phase(const mgrit_level_desc *L, const mgrit_phase_args *A, int32_t *status, cudaStream_t st);
int cl_sweep(const mgrit_level_desc *L, double *U, int64_t ldu, const double *G, int64_t ldg, int zero_init,
             int32_t *gmres_iters, int32_t *status, cudaStream_t st);

int apply_rows_2d(const mgrit_level_desc *L, const RowsArgs &r, void *scratch, int64_t scratch_bytes,
                  int32_t *status, cudaStream_t st);
int level_phase_2d(const mgrit_level_desc *L, const mgrit_phase_args *A, void *scratch, int64_t scratch_bytes,
                   int32_t *status, cudaStream_t st);
int sweep_2d(const mgrit_level_desc *L, double *U, int64_t ldu, const double *G, int64_t ldg, int zero_init,
             int32_t *gmres_iters, void *scratch, int64_t scratch_bytes, int32_t *status, cudaStream_t st);
int records_separable_2d(int32_t n_x, int64_t n_sets, const double *s_x, const double *s_y, int32_t *flag,
                         cudaStream_t st);
int64_t scratch2d_bytes(const mgrit_level_desc *L, int64_t rows);
int64_t capacity2d(const mgrit_level_desc *L);
int axpy_rows_impl(double *U, int64_t ldu, int64_t stride, const double *X, int64_t ldx, int64_t rows,
                   int64_t n, cudaStream_t st);

}  // namespace mgrit
