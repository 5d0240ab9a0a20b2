// step1d_cl.cu — launch policy of the cluster-split corrected steps
// (step1d_cluster.cuh); kernels instantiated in step1d_cl_p{1,3,5}.cu.
#include <type_traits>

#include "step1d_cluster.cuh"

namespace mgrit {

// instantiated in step1d_cl_p{1,3,5}.cu
extern template struct cl::LaunchCl<1>;
extern template struct cl::LaunchCl<3>;
extern template struct cl::LaunchCl<5>;

namespace {

template <typename F>
int by_p(int p, F &&f) {
    switch (p) {
        case 1: return f(cl::LaunchCl<1>{});
        case 3: return f(cl::LaunchCl<3>{});
        default: return f(cl::LaunchCl<5>{});
    }
}

// Cost of a wave of one-CTA corrected steps over a wave of cluster steps
// (x10), measured on B200 per row length: n = 4096 (cfg2 levels 2-5: 0.167 vs
// 0.096 ms per FC phase) and n = 16384 (cfg3 levels 1-3: 0.745 vs 0.142 ms
// per wave); the shorter rows are extrapolated.  Cluster kernels are picked
// when their wave count is below that multiple of the one-CTA kernel's.
int64_t cta_over_cluster10(int n) {
    if (n <= 2048) return 15;
    if (n <= 4096) return 17;
    if (n <= 8192) return 30;
    return 50;
}

}  // namespace

// -1: not taken (caller uses the one-CTA kernels)
int cl_level_phase(const mgrit_level_desc *L, const mgrit_phase_args *A, int32_t *status, cudaStream_t st) {
    if (L->launch_policy == MGRIT_LAUNCH_CTA || !cl::cl_eligible(L)) return -1;
    if (!cl::cl_aligned(A->U) || (A->ldu & 1) || !cl::cl_aligned(A->Cbuf)) return -1;
    if (A->c_count <= 0) return -1;
    const int res_cl = by_p(L->p, [&](auto X) { return decltype(X)::resident_clusters(L); });
    if (res_cl < 1) return -1;
    if (L->launch_policy != MGRIT_LAUNCH_CLUSTER) {
        const int64_t res_cta = rows_capacity(L);
        const int64_t waves_cta = (A->c_count + res_cta - 1) / (res_cta > 0 ? res_cta : 1);
        const int64_t waves_cl = (A->c_count + res_cl - 1) / res_cl;
        if (10 * waves_cl >= cta_over_cluster10(L->n_x) * waves_cta) return -1;
    }
    return by_p(L->p, [&](auto X) { return decltype(X)::phase(L, A, status, st, res_cl); });
}

int cl_sweep(const mgrit_level_desc *L, double *U, int64_t ldu, const double *G, int64_t ldg, int zero_init,
             int32_t *gmres_iters, int32_t *status, cudaStream_t st) {
    if (L->launch_policy == MGRIT_LAUNCH_CTA || !cl::cl_eligible(L)) return -1;
    if (!cl::cl_aligned(U) || (ldu & 1)) return -1;
    return by_p(L->p, [&](auto X) { return decltype(X)::sweep(L, U, ldu, G, ldg, zero_init, gmres_iters, status, st); });
}

}  // namespace mgrit
