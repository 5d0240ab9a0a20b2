// step1d.cu — dispatch of the 1D entry points onto the (P, KIND)
// instantiation units (step1d_p*_k*.cu).
#include <type_traits>

#include "step1d_kernels.cuh"

namespace mgrit {

template <typename F>
static int dispatch_pk(int p, int kind, F &&f) {
    auto by_kind = [&](auto P) {
        constexpr int PP = decltype(P)::value;
        switch (kind) {
            case MGRIT_KIND_SL: return f(Launch1D<PP, MGRIT_KIND_SL>{});
            case MGRIT_KIND_CORRECTED: return f(Launch1D<PP, MGRIT_KIND_CORRECTED>{});
            default: return f(Launch1D<PP, MGRIT_KIND_FORWARD_EULER>{});
        }
    };
    switch (p) {
        case 1: return by_kind(std::integral_constant<int, 1>{});
        case 3: return by_kind(std::integral_constant<int, 3>{});
        default: return by_kind(std::integral_constant<int, 5>{});
    }
}

int64_t rows_capacity(const mgrit_level_desc *L) {
    if (validate(L)) return 0;
    return dispatch_pk(L->p, L->kind, [&](auto X) { return (int)decltype(X)::capacity(L, false); });
}

int64_t rows_capacity_one(const mgrit_level_desc *L) {
    if (validate(L)) return 0;
    return dispatch_pk(L->p, L->kind, [&](auto X) { return (int)decltype(X)::capacity(L, true); });
}

int apply_rows_1d(const mgrit_level_desc *L, const RowsArgs &a, void *scratch,
                  int64_t scratch_bytes, int32_t *status, cudaStream_t st) {
    if (int rc = validate(L)) return rc;
    return dispatch_pk(L->p, L->kind, [&](auto X) {
        return decltype(X)::rows(L, a, scratch, scratch_bytes, status, st);
    });
}

int level_phase_1d(const mgrit_level_desc *L, const mgrit_phase_args *A, void *scratch,
                   int64_t scratch_bytes, int32_t *status, cudaStream_t st) {
    if (int rc = validate(L)) return rc;
    if (L->kind == MGRIT_KIND_CORRECTED && A && A->m >= 1 && A->U && A->Cbuf && A->n_intervals >= 1 &&
        (int64_t)A->n_intervals * A->m == L->n_steps && A->phase >= 0 && A->phase <= 3 &&
        (A->phase != MGRIT_PHASE_INJ_F || A->Uc)) {
        const int rc = cl_level_phase(L, A, status, st);
        if (rc >= 0) return rc;
    }
    return dispatch_pk(L->p, L->kind, [&](auto X) {
        return decltype(X)::phase(L, A, scratch, scratch_bytes, status, st);
    });
}

int sweep_1d(const mgrit_level_desc *L, double *U, int64_t ldu, const double *G, int64_t ldg,
             int zero_init, int32_t *gmres_iters, void *scratch, int64_t scratch_bytes,
             int32_t *status, cudaStream_t st) {
    if (int rc = validate(L)) return rc;
    if ((L->kind == MGRIT_KIND_CORRECTED || L->kind == MGRIT_KIND_SL) && U) {
        const int rc = cl_sweep(L, U, ldu, G, ldg, zero_init, gmres_iters, status, st);
        if (rc >= 0) return rc;
    }
    return dispatch_pk(L->p, L->kind, [&](auto X) {
        return decltype(X)::sweep(L, U, ldu, G, ldg, zero_init, gmres_iters, scratch,
                                  scratch_bytes, status, st);
    });
}

}  // namespace mgrit
