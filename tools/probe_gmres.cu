// Standalone clock64 probe of one corrected step (SL + fixed-K GMRES) in one CTA.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -fmad=false
//      --expt-relaxed-constexpr -DMGRIT_PROBE -o probe tools/probe_gmres.cu
#define MGRIT_LAUNCH1D_IMPL
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../paper_2203_13382_b200/csrc/step1d_kernels.cuh"

namespace mgrit {
void set_error(const char *what, cudaError_t e) { fprintf(stderr, "%s: %s\n", what, cudaGetErrorString(e)); }
int check_launch(const char *what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) { set_error(what, e); return MGRIT_ECUDA; }
    return MGRIT_OK;
}
}  // namespace mgrit
using namespace mgrit;

int main(int argc, char **argv) {
    const int n = argc > 1 ? atoi(argv[1]) : 4096;
    const int K = argc > 2 ? atoi(argv[2]) : 10;
    std::vector<double> s(n), sig(n), u(n);
    srand(1);
    for (int i = 0; i < n; ++i) {
        s[i] = i + 0.37 + 0.2 * (rand() / (double)RAND_MAX);
        if (s[i] >= n) s[i] -= n;
        sig[i] = 0.3 * (rand() / (double)RAND_MAX);
        u[i] = rand() / (double)RAND_MAX;
    }
    double *ds, *dsig, *du, *dout, *scr;
    int *st;
    cudaMalloc(&ds, n * 8); cudaMalloc(&dsig, n * 8); cudaMalloc(&du, n * 8); cudaMalloc(&dout, n * 8);
    cudaMalloc(&scr, (size_t)(K + 1) * n * 8); cudaMalloc(&st, 4); cudaMemset(st, 0, 4);
    cudaMemcpy(ds, s.data(), n * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(dsig, sig.data(), n * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(du, u.data(), n * 8, cudaMemcpyHostToDevice);
    mgrit_level_desc L{};
    L.dim = 1; L.n_x = n; L.p = 3; L.kind = MGRIT_KIND_CORRECTED; L.shared = 1; L.n_steps = 1; L.n_points = n;
    L.s_x = ds; L.sig_x = dsig; L.gmres_max_iters = K; L.gmres_tol = -1.0;
    L.gmres_lowsync = argc > 3 ? atoi(argv[3]) : 0;
    RowsArgs a{1, nullptr, 0, 0, du, n, nullptr, n, nullptr, n, dout, n, nullptr, nullptr};
    for (int rep = 0; rep < 3; ++rep)
        Launch1D<3, MGRIT_KIND_CORRECTED>::rows(&L, a, scr, (int64_t)(K + 1) * n * 8, st, 0);
    cudaDeviceSynchronize();
    long long h[512];
    cudaMemcpyFromSymbol(h, g_probe, sizeof(h));
    printf("n=%d K=%d  SL %lld  beta %lld\n", n, K, h[1] - h[0], h[2] - h[1]);
    for (int kk = 0; kk < K; ++kk) {
        long long *q = h + 10 + 8 * kk;
        printf(" kk=%d stencil %5lld  MGS(%d) %6lld (%5lld/step)  norm %5lld  normalize %5lld  givens %5lld  sync %5lld  total %6lld\n",
               kk, q[1] - q[0], kk + 1, q[2] - q[1], (q[2] - q[1]) / (kk + 1), q[3] - q[2], q[4] - q[3], q[5] - q[4],
               q[6] - q[5], q[6] - q[0]);
    }
    printf(" xcomb %lld   total %lld cycles\n", h[201] - h[200], h[201] - h[0]);
    if (K > 5 && L.gmres_lowsync)
        printf("  kk=5 lowsync: passA %lld  bar %lld  warp0 %lld  bar %lld  passB %lld\n", h[302] - h[301],
               h[303] - h[302], h[304] - h[303], h[305] - h[304], h[306] - h[305]);
    else if (K > 5)
        for (int j = 0; j <= 5; ++j) {
            long long *q = h + 300 + 4 * j;
            printf("  kk=5 j=%d: dot->prefetch-issued %lld, prefetch->h %lld (reduction), h->axpy-done %lld, next-dot %lld\n",
                   j, q[1] - q[0], q[2] - q[1], q[3] - q[2], j < 5 ? q[4] - q[3] : 0LL);
        }
    return 0;
}
