// common.cuh — device building blocks shared by all MGRIT kernels (sm_100a).
//
// Arithmetic that must be bit-identical to the reference is written with
// explicit round-to-nearest intrinsics (__dmul_rn/__dadd_rn/__dsub_rn) and
// the whole library is compiled with -fmad=false, so no FMA contraction can
// change rounding.  FMA is used only where it is part of an exact algorithm
// (the constant-divisor correction in lagrange_weights).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/mgrit_b200.h"

namespace mgrit {

constexpr double kXLo = -1.0;
constexpr double kLen = 2.0;

// ---------------------------------------------------------------------------
// periodic decomposition (semi_lagrangian.py:118-137)

// s = mod(x - x_lo, L) / h with numpy's float remainder semantics
// (fmod, then += L when the signs differ, +0 when zero).
__device__ __forceinline__ double scaled_coord(double x, double h) {
    double d = __dsub_rn(x, kXLo);
    double r = fmod(d, kLen);
    if (r != 0.0) {
        if (r < 0.0) r = __dadd_rn(r, kLen);
    } else {
        r = 0.0;
    }
    return __ddiv_rn(r, h);
}

struct Dec {
    int e;       // east index in [0, n)
    double eps;  // offset in [0, 1)
};

// east = ceil(s), eps = east - s, rounding guards, east mod n.
// s = mod(x - x_lo, L)/h lies in [0, n], so east in [-1, n] before the
// periodic wrap: two compares instead of an integer division.  ceil and the
// int conversion avoid the low-throughput XU pipe (FRND / F2I): for
// 0 <= s < 2^52, t = s + 2^52 rounds s to the nearest integer r, exactly
// stored in t's low mantissa bits; ceil(s) = r or r + 1.  Same bits as ceil().
__device__ __forceinline__ Dec decompose_s(double s, int n) {
    const double t = __dadd_rn(s, 4503599627370496.0);  // 2^52
    int e = __double2loint(t);
    double ef = __dsub_rn(t, 4503599627370496.0);        // exact: nearest integer to s
    if (ef < s) {
        ef = __dadd_rn(ef, 1.0);
        e += 1;
    }
    // ef = ceil(s) >= s, so RN(ef - s) >= 0: the reference's "eps < 0 -> 0"
    // guard (semi_lagrangian.py:131) can never fire here and is omitted
    double eps = __dsub_rn(ef, s);
    if (eps >= 1.0) {
        eps = __dsub_rn(eps, 1.0);
        e -= 1;
    }
    if (e >= n) e -= n;
    if (e < 0) e += n;
    Dec d;
    d.e = e;
    d.eps = eps;
    return d;
}

// ---------------------------------------------------------------------------
// Lagrange weights (semi_lagrangian.py:140-161).
// w_j = prod_{q != j}(z - q) / prod_{q != j}(j - q), z = -eps, offsets -l..r.
// The division by the integer denominator D uses q0 = num*(1/D),
// r = fma(-q0, D, num) (exact), q = fma(r, 1/D, q0): with 1/D correctly
// rounded this is the correctly rounded quotient (Markstein), i.e. identical
// to num / D; verified over 2e8 random operands and by the GPU parity tests.

template <int P>
struct Stencil {
    static constexpr int L = (P + 1) / 2;  // west extent
    static constexpr int R = (P - 1) / 2;  // east extent
    static constexpr int Q = P + 1;        // taps
};

template <int P>
__device__ __forceinline__ double lagrange_den(int col) {
    constexpr int L = Stencil<P>::L, R = Stencil<P>::R;
    double den = 1.0;
    int j = col - L;
#pragma unroll
    for (int q = -L; q <= R; ++q)
        if (q != j) den *= (double)(j - q);
    return den;
}

__device__ __forceinline__ double div_const(double num, double den, double inv) {
    double q0 = __dmul_rn(num, inv);
    double r = fma(-q0, den, num);
    return fma(r, inv, q0);
}

// a / b with y = RN(1/b): q0 = RN(a y), r = fma(-q0, b, a) (exact),
// q = fma(r, y, q0) == RN(a / b) (Markstein; verified on 4e8 random pairs).
__device__ __forceinline__ double div_rcp(double a, double b, double y) {
    const double q0 = __dmul_rn(a, y);
    const double r = fma(-q0, b, a);
    return fma(r, y, q0);
}

template <int P>
__device__ __forceinline__ void lagrange_weights(double eps, double (&w)[P + 1]) {
    constexpr int L = Stencil<P>::L, R = Stencil<P>::R;
    const double z = -eps;
#pragma unroll
    for (int col = 0; col <= P; ++col) {
        const int j = col - L;
        // num = ((1 * (z - q0)) * (z - q1)) * ...; 1 * x == x exactly
        double num = 0.0;
        bool first = true;
#pragma unroll
        for (int q = -L; q <= R; ++q) {
            if (q == j) continue;
            const double f = q == 0 ? z : __dsub_rn(z, (double)q);  // z - 0 == z exactly
            num = first ? f : __dmul_rn(num, f);
            first = false;
        }
        const double den = lagrange_den<P>(col);
        const double ad = den < 0 ? -den : den;
        if (ad == 1.0 || ad == 2.0 || ad == 4.0 || ad == 8.0 || ad == 16.0)
            w[col] = __dmul_rn(num, 1.0 / den);  // power-of-two denominator: exact
        else
            w[col] = div_const(num, den, 1.0 / den);
    }
}

// ---------------------------------------------------------------------------
// truncation-error polynomial f(z) = prod_{q=-l}^{r}(q + z) / (p+1)!
// (coarse_correction.py:22-32) — setup only, true division.
template <int P>
__device__ __forceinline__ double f_poly(double z) {
    constexpr int L = Stencil<P>::L, R = Stencil<P>::R;
    double out = 1.0;
#pragma unroll
    for (int q = -L; q <= R; ++q) out = __dmul_rn(out, __dadd_rn((double)q, z));
    double fact = 1.0;
#pragma unroll
    for (int k = 2; k <= P + 1; ++k) fact *= (double)k;
    return __ddiv_rn(out, fact);
}

// D_{p+1} stencil coefficients (coarse_correction.py:35-47)
template <int P>
__device__ __forceinline__ double dcoef(int idx);
template <>
__device__ __forceinline__ double dcoef<1>(int i) {
    const double c[3] = {1.0, -2.0, 1.0};
    return c[i];
}
template <>
__device__ __forceinline__ double dcoef<3>(int i) {
    const double c[5] = {1.0, -4.0, 6.0, -4.0, 1.0};
    return c[i];
}
template <>
__device__ __forceinline__ double dcoef<5>(int i) {
    const double c[7] = {1.0, -6.0, 15.0, -20.0, 15.0, -6.0, 1.0};
    return c[i];
}

// c_idx * x for the D stencil; the +-1 coefficients are applied exactly
// without a multiply (1 * x == x, -1 * x == -x in IEEE arithmetic)
template <int P>
__device__ __forceinline__ double cmul(int idx, double x) {
    const double c = dcoef<P>(idx);
    if (c == 1.0) return x;
    if (c == -1.0) return -x;
    return __dmul_rn(c, x);
}

// ---------------------------------------------------------------------------
// deterministic reductions

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = __dadd_rn(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;  // identical in every lane (commutative butterfly)
}

// Block-wide sum; `red` needs NT/32 + 1 doubles of shared memory.  Fixed
// order: per-warp butterfly, then warp 0 sums the warp partials.  Ends with a
// barrier so `red` can be reused immediately.
template <int NT>
__device__ __forceinline__ double block_sum(double v, double *red) {
    constexpr int NW = NT / 32;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    v = warp_sum(v);
    if (lane == 0) red[warp] = v;
    __syncthreads();
    if (warp == 0) {
        double t = lane < NW ? red[lane] : 0.0;
        t = warp_sum(t);
        if (lane == 0) red[NW] = t;
    }
    __syncthreads();
    double r = red[NW];
    __syncthreads();
    return r;
}

// ---------------------------------------------------------------------------
// wave speeds (core.py:130-153 + BASELINE B2/B4).  Expression order follows
// oracle/mgrit_oracle.py:SPEEDS; only sin/cos differ from numpy (<= ulps).

constexpr double kPi = 3.141592653589793;
constexpr double kTwoPi = 2.0 * kPi;  // == Python 2.0 * np.pi (exact doubling)

__device__ __forceinline__ void wave_speed(int id, double x, double y, double t,
                                           double &ax, double &ay) {
    switch (id) {
        case MGRIT_SPEED_C1: ax = 1.0; ay = 0.0; break;
        case MGRIT_SPEED_C2: ax = __dmul_rn(cos(__dmul_rn(kTwoPi, t)), 1.0); ay = 0.0; break;
        case MGRIT_SPEED_C3:
            ax = __dmul_rn(cos(__dmul_rn(kTwoPi, t)), cos(__dmul_rn(kTwoPi, x)));
            ay = 0.0;
            break;
        case MGRIT_SPEED_C4: ax = 1.0; ay = 1.0; break;
        case MGRIT_SPEED_C5: {
            double ct = cos(__ddiv_rn(__dmul_rn(kTwoPi, t), 3.4));
            double sy = sin(__dmul_rn(kPi, y));
            double cx = cos(__dmul_rn(kPi, x));
            ax = __dmul_rn(__dmul_rn(sy, sy), ct);
            ay = __dmul_rn(-__dmul_rn(cx, cx), ct);
            break;
        }
        case MGRIT_SPEED_B2:
            ax = __dadd_rn(1.0, __dmul_rn(__dmul_rn(0.5, sin(__dmul_rn(kTwoPi, x))),
                                         cos(__dmul_rn(kTwoPi, t))));
            ay = 0.0;
            break;
        case MGRIT_SPEED_B4: {
            double ct = cos(__dmul_rn(kTwoPi, t));
            double cx = cos(__dmul_rn(kPi, x));
            double sy = sin(__dmul_rn(kPi, y));
            ax = __dadd_rn(__dmul_rn(__dmul_rn(cx, cx), ct), 0.5);
            ay = __dadd_rn(__dmul_rn(__dmul_rn(sy, sy), ct), 0.5);
            break;
        }
        default: ax = 0.0; ay = 0.0; break;
    }
}

// ---------------------------------------------------------------------------
// error plumbing

void set_error(const char *what, cudaError_t e);
int check_launch(const char *what);

}  // namespace mgrit
