// Standalone timing probe of the cooperative 2D GMRES (tools only): globaltimer
// stamps of every CTA at every system barrier of one gmres2d_coop launch.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -fmad=false --expt-relaxed-constexpr \
//        -DMGRIT_PROBE2D -o tools/probe_coop2d tools/probe_coop2d.cu
//   ./tools/probe_coop2d [n_x=1024] [p=5] [K=4] [systems=4]
// Synthetic separable-ish records (CFL ~ 6 shifts), sigma ~ 0.05, fixed K Arnoldi steps.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_2203_13382_b200/csrc/step2d.cu"

namespace mgrit {
static char g_err[256];
void set_error(const char *what, cudaError_t e) { snprintf(g_err, sizeof g_err, "%s: %s", what, cudaGetErrorString(e)); fprintf(stderr, "%s\n", g_err); }
int check_launch(const char *what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) { set_error(what, e); return MGRIT_ECUDA; }
    return MGRIT_OK;
}
// (capi.cu's row add is not needed by the probe)
int axpy_rows_impl(double *, int64_t, int64_t, const double *, int64_t, int64_t, int64_t, cudaStream_t) { return MGRIT_EINVAL; }
}  // namespace mgrit
using namespace mgrit;

int main(int argc, char **argv) {
    const int nx = argc > 1 ? atoi(argv[1]) : 1024, p = argc > 2 ? atoi(argv[2]) : 5, K = argc > 3 ? atoi(argv[3]) : 4;
    const int B = argc > 4 ? atoi(argv[4]) : 4;
    const int64_t n = (int64_t)nx * nx;
    std::vector<double> sx(n), sy(n), gx(n), gy(n), u((size_t)B * n);
    srand(1);
    auto rnd = [] { return rand() / (double)RAND_MAX; };
    for (int iy = 0; iy < nx; ++iy)
        for (int ix = 0; ix < nx; ++ix) {
            const int64_t i = (int64_t)iy * nx + ix;
            double a = ix - 6.3 - 3.0 * cos(6.283185307179586 * ix / nx) + 1e-9 * rnd();
            double b = iy - 5.7 - 3.0 * sin(6.283185307179586 * iy / nx) + 1e-9 * rnd();
            sx[i] = fmod(a + nx, (double)nx);
            sy[i] = fmod(b + nx, (double)nx);
            gx[i] = 0.05 * rnd();
            gy[i] = 0.05 * rnd();
        }
    for (auto &v : u) v = rnd();
    double *dsx, *dsy, *dgx, *dgy, *du, *dout;
    int *st;
    cudaMalloc(&dsx, n * 8); cudaMalloc(&dsy, n * 8); cudaMalloc(&dgx, n * 8); cudaMalloc(&dgy, n * 8);
    cudaMalloc(&du, (size_t)B * n * 8); cudaMalloc(&dout, (size_t)B * n * 8); cudaMalloc(&st, 4); cudaMemset(st, 0, 4);
    cudaMemcpy(dsx, sx.data(), n * 8, cudaMemcpyHostToDevice); cudaMemcpy(dsy, sy.data(), n * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(dgx, gx.data(), n * 8, cudaMemcpyHostToDevice); cudaMemcpy(dgy, gy.data(), n * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(du, u.data(), (size_t)B * n * 8, cudaMemcpyHostToDevice);
    mgrit_level_desc L{};
    L.dim = 2; L.n_x = nx; L.p = p; L.kind = MGRIT_KIND_CORRECTED; L.shared = 1; L.n_steps = 1; L.n_points = n;
    L.s_x = dsx; L.s_y = dsy; L.sig_x = dgx; L.sig_y = dgy; L.gmres_max_iters = K; L.gmres_tol = -1.0;
    const int64_t rows = std::min<int64_t>(B, capacity2d(&L));
    const int64_t sbytes = scratch2d_bytes(&L, rows);
    void *scr;
    cudaMalloc(&scr, sbytes);
    const int ctas = 148 * 4;
    unsigned long long *probe;
    cudaMalloc(&probe, (size_t)ctas * kProbeBars * 2 * 8);
    RowsArgs a{B, nullptr, 0, 0, du, n, nullptr, n, nullptr, n, dout, n, nullptr, nullptr};
    for (int rep = 0; rep < 2; ++rep) apply_rows_2d(&L, a, scr, sbytes, st, 0);   // warm
    cudaDeviceSynchronize();
    cudaMemset(probe, 0, (size_t)ctas * kProbeBars * 2 * 8);
    cudaMemcpyToSymbol(g_probe2d, &probe, sizeof(probe));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    apply_rows_2d(&L, a, scr, sbytes, st, 0);
    cudaEventRecord(e1);
    cudaDeviceSynchronize();
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    std::vector<unsigned long long> h((size_t)ctas * kProbeBars * 2);
    cudaMemcpy(h.data(), probe, h.size() * 8, cudaMemcpyDeviceToHost);
    const int chunks = ctas / (int)rows;
    printf("n_x=%d p=%d K=%d systems=%d rows in flight=%lld chunks=%d launch %.1f us (%.1f us per system-slot pass)\n", nx, p, K, B,
           (long long)rows, chunks, ms * 1e3, ms * 1e3 / ((B + rows - 1) / rows));
    // slot 0: CTAs 0 .. chunks-1
    unsigned long long t0 = ~0ull;
    for (int c = 0; c < chunks; ++c) t0 = std::min(t0, h[((size_t)c * kProbeBars) * 2]);
    printf("barrier: first arrival, median arrival, last arrival, median release (us since the slot's first stamp); interval = last arrival - previous release\n");
    double prev_rel = 0;
    for (int g = 0; g < kProbeBars; ++g) {
        std::vector<double> arr, rel;
        for (int c = 0; c < chunks; ++c) {
            const unsigned long long ta = h[((size_t)c * kProbeBars + g) * 2], tr = h[((size_t)c * kProbeBars + g) * 2 + 1];
            if (ta) { arr.push_back((ta - t0) * 1e-3); rel.push_back((tr - t0) * 1e-3); }
        }
        if (arr.empty()) break;
        std::sort(arr.begin(), arr.end()); std::sort(rel.begin(), rel.end());
        printf(" #%2d  arrive %8.2f %8.2f %8.2f   release %8.2f   pass(first) %6.2f  pass(last) %6.2f  skew %6.2f  barrier %5.2f\n", g, arr.front(), arr[arr.size() / 2],
               arr.back(), rel[rel.size() / 2], arr.front() - prev_rel, arr.back() - prev_rel, arr.back() - arr.front(), rel[rel.size() / 2] - arr.back());
        prev_rel = rel[rel.size() / 2];
    }
    return 0;
}
