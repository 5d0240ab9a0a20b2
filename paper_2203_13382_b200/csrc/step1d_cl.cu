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

// A one-CTA corrected step costs about 1.7x a cluster step (B200, n = 4096,
// cfg2 levels 3-5: 0.167 vs 0.096 ms per FC phase); pick the cluster kernels
// when their wave count is below 1.7x the one-CTA kernel's.
constexpr int64_t kCtaOverCluster10 = 17;

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
        if (10 * waves_cl >= kCtaOverCluster10 * waves_cta) return -1;
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
