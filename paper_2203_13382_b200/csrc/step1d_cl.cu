// step1d_cl.cu — launch policy of the cluster-split corrected steps
// (step1d_cluster.cuh); kernels instantiated in step1d_cl_p{1,3,5}_cs{2,4,8,16}.cu.
#include <type_traits>

#include "step1d_cluster.cuh"

namespace mgrit {

#define MGRIT_CL_EXTERN(P)                        \
    extern template struct cl::LaunchCl<P, 2>;  \
    extern template struct cl::LaunchCl<P, 4>;  \
    extern template struct cl::LaunchCl<P, 8>;  \
    extern template struct cl::LaunchCl<P, 16>;
MGRIT_CL_EXTERN(1)
MGRIT_CL_EXTERN(3)
MGRIT_CL_EXTERN(5)
#undef MGRIT_CL_EXTERN

namespace {

constexpr int kClSizes[] = {2, 4, 8, 16};

template <typename F>
int by_p_cs(int p, int cs, F &&f) {
    auto by_cs = [&](auto P) {
        constexpr int PP = decltype(P)::value;
        switch (cs) {
            case 2: return f(cl::LaunchCl<PP, 2>{});
            case 4: return f(cl::LaunchCl<PP, 4>{});
            case 16: return f(cl::LaunchCl<PP, 16>{});
            default: return f(cl::LaunchCl<PP, 8>{});
        }
    };
    switch (p) {
        case 1: return by_cs(std::integral_constant<int, 1>{});
        case 3: return by_cs(std::integral_constant<int, 3>{});
        default: return by_cs(std::integral_constant<int, 5>{});
    }
}

bool cs_eligible(const mgrit_level_desc *L, int cs) {
    switch (cs) {
        case 2: return cl::cl_eligible<2>(L);
        case 4: return cl::cl_eligible<4>(L);
        case 16: return cl::cl_eligible<16>(L);
        default: return cl::cl_eligible<8>(L);
    }
}

// MGRIT_LAUNCH_CLUSTER{2,4,8,16}: one fixed cluster size (tests, measurement)
int forced_cs(const mgrit_level_desc *L) {
    switch (L->launch_policy) {
        case MGRIT_LAUNCH_CLUSTER2: return 2;
        case MGRIT_LAUNCH_CLUSTER4: return 4;
        case MGRIT_LAUNCH_CLUSTER8: return 8;
        case MGRIT_LAUNCH_CLUSTER16: return 16;
        default: return 0;
    }
}

// Time of one wave of cluster steps relative to one wave of one-CTA steps
// (x100), per cluster size and row length, measured on B200 with
// tools/gpu_cluster_sizes.sh (V-cycle phases of cfg1_085h / cfg2 / cfg3 with
// every corrected level forced to one shape; profiles/r01_cluster_sizes.jsonl):
//   n = 1024  (cfg1_085h 128-step sweep): CTA 3.59 ms, CS 2/4/8: 2.97/2.99/3.11
//   n = 4096  (cfg2 level 4, 4 chains, one wave each): CTA 0.532 ms,
//             CS 2/4/8/16: 0.472/0.346/0.332/0.341
//   n = 16384 (cfg3 levels 1-4): CS 8 ~17, CS 16 ~8 per wave vs the CTA wave
// 0 = not measured (not used by the automatic policy).
int cl_wave_cost100(int cs, int n) {
    if (n <= 2048) {
        switch (cs) { case 2: return 83; case 4: return 84; case 8: return 87; default: return 0; }
    }
    if (n <= 4096) {
        switch (cs) { case 2: return 89; case 4: return 65; case 8: return 62; default: return 64; }
    }
    if (n <= 8192) return cs == 8 ? 33 : 0;
    switch (cs) { case 8: return 17; case 16: return 8; default: return 0; }
}

int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / (b > 0 ? b : 1); }

int cl_resident(const mgrit_level_desc *L, int cs) {
    return by_p_cs(L->p, cs, [&](auto X) { return decltype(X)::resident_clusters(L); });
}

}  // namespace

// -1: not taken (caller uses the one-CTA kernels)
int cl_level_phase(const mgrit_level_desc *L, const mgrit_phase_args *A, int32_t *status, cudaStream_t st) {
    if (L->launch_policy == MGRIT_LAUNCH_CTA) return -1;
    if (!cl::cl_aligned(A->U) || (A->ldu & 1) || !cl::cl_aligned(A->Cbuf)) return -1;
    if (A->c_count <= 0) return -1;
    const int force = forced_cs(L);
    int best_cs = 0, best_res = 0;
    int64_t best_cost = -1;
    // one-CTA cost in units of 1/100 wave (two-CTAs-per-SM waves cost 1.66)
    int64_t cta_cost = -1;
    if (L->launch_policy != MGRIT_LAUNCH_CLUSTER && !force) {
        const int64_t res_cta = rows_capacity(L);
        const int64_t res_one = rows_capacity_one(L);
        cta_cost = A->c_count <= res_one ? 100
                   : (res_cta > res_one && L->launch_policy != MGRIT_LAUNCH_AUTO_ONE)
                       ? ceil_div(A->c_count, res_cta) * 166
                       : ceil_div(A->c_count, res_one) * 100;
    }
    for (int cs : kClSizes) {
        if (force && cs != force) continue;
        if (!cs_eligible(L, cs)) continue;
        const int w = cl_wave_cost100(cs, L->n_x);
        if (!force && w == 0) continue;
        const int res = cl_resident(L, cs);
        if (res < 1) continue;
        const int64_t cost = ceil_div(A->c_count, res) * (w ? w : 1);
        if (best_cost < 0 || cost < best_cost) {
            best_cost = cost;
            best_cs = cs;
            best_res = res;
        }
    }
    if (!best_cs) return -1;
    if (cta_cost >= 0 && !force && best_cost >= cta_cost) return -1;
    return by_p_cs(L->p, best_cs, [&](auto X) { return decltype(X)::phase(L, A, status, st, best_res); });
}

int cl_sweep(const mgrit_level_desc *L, double *U, int64_t ldu, const double *G, int64_t ldg, int zero_init,
             int32_t *gmres_iters, int32_t *status, cudaStream_t st) {
    if (L->launch_policy == MGRIT_LAUNCH_CTA) return -1;
    if (!cl::cl_aligned(U) || (ldu & 1)) return -1;
    // one chain: the size with the cheapest wave
    const int force = forced_cs(L);
    int best_cs = 0, best_w = 0;
    if (L->kind == MGRIT_KIND_SL) {
        // plain SL sweep (sequential time stepping of a fine level): only on
        // request (MGRIT_LAUNCH_CLUSTER*), the largest eligible cluster
        if (L->launch_policy != MGRIT_LAUNCH_CLUSTER && !force) return -1;
        for (int cs : kClSizes)
            if ((!force || cs == force) && cs_eligible(L, cs)) best_cs = cs;
        if (!best_cs) return -1;
        return by_p_cs(L->p, best_cs, [&](auto X) {
            return decltype(X)::sweep(L, U, ldu, G, ldg, zero_init, gmres_iters, status, st);
        });
    }
    for (int cs : kClSizes) {
        if (force && cs != force) continue;
        if (!cs_eligible(L, cs)) continue;
        const int w = cl_wave_cost100(cs, L->n_x);
        if (!force && w == 0) continue;
        if (!best_cs || (w && w < best_w)) {
            best_cs = cs;
            best_w = w;
        }
    }
    if (!best_cs) return -1;
    return by_p_cs(L->p, best_cs, [&](auto X) {
        return decltype(X)::sweep(L, U, ldu, G, ldg, zero_init, gmres_iters, status, st);
    });
}

}  // namespace mgrit
