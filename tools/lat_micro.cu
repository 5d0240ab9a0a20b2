// dependent-chain latencies (cycles/op) of FP64 and shuffle ops on this GPU
#include <cstdio>
__global__ void k(double *out, long long *cyc, double a, double b) {
    double x = a;
    int lane = threadIdx.x;
    long long t0 = clock64();
#pragma unroll
    for (int i = 0; i < 100; ++i) { x = __dadd_rn(x, b); }
    long long t1 = clock64();
#pragma unroll
    for (int i = 0; i < 100; ++i) { x = fma(x, a, b); }
    long long t2 = clock64();
#pragma unroll
    for (int i = 0; i < 100; ++i) { x = __shfl_xor_sync(0xffffffffu, x, 1); }
    long long t3 = clock64();
    float f = (float)x;
#pragma unroll
    for (int i = 0; i < 100; ++i) { f = fmaf(f, 1.0001f, 0.5f); }
    long long t4 = clock64();
#pragma unroll
    for (int i = 0; i < 100; ++i) { x = __dadd_rn(x, __shfl_xor_sync(0xffffffffu, x, 1)); }
    long long t5 = clock64();
#pragma unroll
    for (int i = 0; i < 100; ++i) { x = __drcp_rn(x + 1.0); }
    long long t6 = clock64();
#pragma unroll
    for (int i = 0; i < 100; ++i) { x = __ddiv_rn(b, x + 1.0); }
    long long t7 = clock64();
#pragma unroll
    for (int i = 0; i < 100; ++i) { x = hypot(x, b); }
    long long t8 = clock64();
    out[lane] = x + f;
    if (lane == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4; cyc[5] = t6 - t5; cyc[6] = t7 - t6; cyc[7] = t8 - t7; }
}
int main() {
    double *o; long long *c, h[8];
    cudaMalloc(&o, 256); cudaMalloc(&c, 64);
    for (int r = 0; r < 2; ++r) k<<<1, 32>>>(o, c, 1.000001, 0.5);
    cudaMemcpy(h, c, 64, cudaMemcpyDeviceToHost);
    const char *nm[8] = {"dadd", "dfma", "shfl.f64", "ffma", "dadd+shfl", "drcp", "ddiv", "hypot"};
    for (int i = 0; i < 8; ++i) printf("%-10s %6.1f cyc/op\n", nm[i], h[i] / 100.0);
}
