// clock64 probe of the cluster-split corrected step (rank 0, thread 0):
// one sweep step (SL + fixed-K GMRES) on one 8-CTA cluster.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -fmad=false
//      --expt-relaxed-constexpr -DMGRIT_PROBE -o tools/probe_cluster tools/probe_cluster.cu
#define MGRIT_LAUNCHCL_IMPL
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../paper_2203_13382_b200/csrc/step1d_cluster.cuh"

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
    const int lowsync = argc > 3 ? atoi(argv[3]) : 0;
    const int steps = argc > 4 ? atoi(argv[4]) : 1;
    const int csz = argc > 5 ? atoi(argv[5]) : 8;   // cluster size 2 / 4 / 8 / 16
    std::vector<double> s(n), sig(n), u((steps + 1) * n, 0.0);
    srand(1);
    for (int i = 0; i < n; ++i) {
        s[i] = i + 0.37 + 0.2 * (rand() / (double)RAND_MAX);
        if (s[i] >= n) s[i] -= n;
        sig[i] = 0.3 * (rand() / (double)RAND_MAX);
        u[i] = rand() / (double)RAND_MAX;
    }
    double *ds, *dsig, *du;
    int *st;
    cudaMalloc(&ds, n * 8); cudaMalloc(&dsig, n * 8); cudaMalloc(&du, (steps + 1) * n * 8);
    cudaMalloc(&st, 4); cudaMemset(st, 0, 4);
    cudaMemcpy(ds, s.data(), n * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(dsig, sig.data(), n * 8, cudaMemcpyHostToDevice);
    mgrit_level_desc L{};
    L.dim = 1; L.n_x = n; L.p = 3; L.kind = MGRIT_KIND_CORRECTED; L.shared = 1; L.n_steps = steps; L.n_points = n;
    L.s_x = ds; L.sig_x = dsig; L.gmres_max_iters = K; L.gmres_tol = -1.0; L.gmres_lowsync = lowsync;
    for (int rep = 0; rep < 3; ++rep) {
        cudaMemcpy(du, u.data(), (steps + 1) * n * 8, cudaMemcpyHostToDevice);
        int rc = csz == 2 ? cl::LaunchCl<3, 2>::sweep(&L, du, n, nullptr, 0, 0, nullptr, st, 0)
               : csz == 4 ? cl::LaunchCl<3, 4>::sweep(&L, du, n, nullptr, 0, 0, nullptr, st, 0)
               : csz == 16 ? cl::LaunchCl<3, 16>::sweep(&L, du, n, nullptr, 0, 0, nullptr, st, 0)
                           : cl::LaunchCl<3, 8>::sweep(&L, du, n, nullptr, 0, 0, nullptr, st, 0);
        if (rc) { printf("launch rc %d\n", rc); return 1; }
    }
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
    long long h[512];
    cudaMemcpyFromSymbol(h, g_probe, sizeof(h));
    printf("CS=%d ", csz);
    printf("n=%d K=%d lowsync=%d steps=%d  await_row %lld  SL+sig %lld  beta %lld  b0 %lld\n", n, K, lowsync, steps, h[401] - h[400],
           h[402] - h[401], h[403] - h[402], h[404] - h[403]);
    for (int kk = 0; kk < K; ++kk) {
        long long *q = h + 410 + 6 * kk;
        printf(" kk=%d stencil %5lld  project %6lld  norm %5lld  normalize %5lld  givens+sync %5lld  total %6lld\n", kk,
               q[1] - q[0], q[2] - q[1], q[3] - q[2], q[4] - q[3], q[5] - q[4], q[5] - q[0]);
    }
    printf(" after-loop sync %lld  backsub %lld  sync %lld  xcomb %lld\n", h[482] - h[410 + 6 * (K - 1) + 5],
           h[483] - h[482], h[484] - h[483], h[481] - h[484]);
    printf(" backsub+xcomb %lld   total %lld cycles\n", h[481] - h[410 + 6 * (K - 1) + 5], h[481] - h[400]);
    return 0;
}
