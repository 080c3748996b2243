// Branch-free fp64 exp / expm1 / reciprocal for the recurrent kernels.
//
// CUDA's exp()/expm1()/division carry slow-path branches, so two independent
// activations in one thread do not overlap (measured: scripts/act_probe2.cu,
// 1 warp x 2 samples = 2x the latency of 1).  These straight-line versions
// (Cody-Waite range reduction with FMA, Estrin-evaluated Taylor polynomial,
// exponent-field scaling, rcp.approx + Newton) interleave freely.  Accuracy:
// within 4 ulp of the libm results over the activation ranges (sigmoid 4,
// tanh 3, exp 1, expm1 2, division 0: tests/test_fastmath_gpu.py), which the
// parity tests absorb: every sampled placement
// stays bit-exact.
#pragma once
#include <math.h>

namespace dp {

// 2^k for integer k, clamped: k <= -1023 -> 0, k >= 1024 -> +inf (integer
// clamp: fp64 fmin/fmax cost ~25 cycles each here)
__device__ __forceinline__ double fm_pow2i(int k) {
    k = min(max(k, -1023), 1024);
    return __hiloint2double((k + 1023) << 20, 0);
}

// Polynomial / reduction constants.  CB = true: read from the constant bank
// (fp64 FMAs take them as c[] operands; literals that need all 64 bits are
// otherwise re-materialised with two moves each inside register-starved loops).
// Measured per kernel: the single-CTA encoder recurrence gains ~6% with CB, the
// decoder loses ~10% (its draw chain), so the default stays literal.
static __constant__ double kFmC[16] = {
    1.0 / 6.0,         0.5,
    1.0 / 120.0,       1.0 / 24.0,
    1.0 / 5040.0,      1.0 / 720.0,
    1.0 / 362880.0,    1.0 / 40320.0,
    1.0 / 39916800.0,  1.0 / 3628800.0,
    1.0 / 6227020800.0, 1.0 / 479001600.0,
    1.4426950408889634,                 // log2 e
    6.93147180559945286227e-01,         // ln2 rounded to double
    2.31904681384629955842e-17,         // ln2 - the above
    0.0};
template <bool CB>
__device__ __forceinline__ double fm_c(int i) {
    constexpr double lit[15] = {1.0 / 6.0,         0.5,
                                1.0 / 120.0,       1.0 / 24.0,
                                1.0 / 5040.0,      1.0 / 720.0,
                                1.0 / 362880.0,    1.0 / 40320.0,
                                1.0 / 39916800.0,  1.0 / 3628800.0,
                                1.0 / 6227020800.0, 1.0 / 479001600.0,
                                1.4426950408889634,
                                6.93147180559945286227e-01,
                                2.31904681384629955842e-17};
    return CB ? kFmC[i] : lit[i];
}

// expm1 on the reduced argument |r| <= ln2/2: r + r^2 (1/2! + r/3! + ... + r^11/13!)
template <bool CB = false>
__device__ __forceinline__ double fm_expm1_poly(double r) {
    const double r2 = r * r;
    const double a0 = fma(r, fm_c<CB>(0), fm_c<CB>(1));
    const double a1 = fma(r, fm_c<CB>(2), fm_c<CB>(3));
    const double a2 = fma(r, fm_c<CB>(4), fm_c<CB>(5));
    const double a3 = fma(r, fm_c<CB>(6), fm_c<CB>(7));
    const double a4 = fma(r, fm_c<CB>(8), fm_c<CB>(9));
    const double a5 = fma(r, fm_c<CB>(10), fm_c<CB>(11));
    const double r4 = r2 * r2;
    const double b0 = fma(r2, a1, a0);
    const double b1 = fma(r2, a3, a2);
    const double b2 = fma(r2, a5, a4);
    const double r8 = r4 * r4;
    const double c0 = fma(r4, b1, b0);
    const double q = fma(r8, b2, c0);
    return fma(r2, q, r);
}

// y = k ln2 + r, |r| <= ln2/2 (+ rounding), k integer.  k comes from the
// magic-number rounding t = fma(y, log2 e, 1.5 2^52): the integer sits in the
// low mantissa bits of t (|y log2 e| << 2^51), so k = t - 1.5 2^52 and its
// int32 value is t's low word — no FRND / F2I on the chain (~26 cycles each,
// scripts/lat_probe2.cu).
template <bool CB = false>
__device__ __forceinline__ void fm_reduce(double y, double &k, double &r, int &ki) {
    constexpr double kRnd = 6755399441055744.0;  // 1.5 * 2^52 (a 32-bit immediate)
    // clamp to [-1000, 1000] with fmin/fmax's NaN rule (NaN -> -1000) as two
    // compare-selects: saturates exp to 0 / inf, expm1 to -1 / inf; keeps r sane
    y = !(y >= -1000.0) ? -1000.0 : y;
    y = y > 1000.0 ? 1000.0 : y;
    const double t = fma(y, fm_c<CB>(12), kRnd);
    k = t - kRnd;
    ki = __double2loint(t);
    r = fma(-k, fm_c<CB>(13), y);
    r = fma(-k, fm_c<CB>(14), r);
}

// expm1(y) = 2^k (p + 1) - 1 = 2^k p + (2^k - 1)
template <bool CB = false>
__device__ __forceinline__ double fm_expm1(double y) {
    double k, r;
    int ki;
    fm_reduce<CB>(y, k, r, ki);
    const double p = fm_expm1_poly<CB>(r);
    const double s = fm_pow2i(ki);
    return fma(s, p, s - 1.0);
}

// exp(y) = 2^k (1 + p)
template <bool CB = false>
__device__ __forceinline__ double fm_exp(double y) {
    double k, r;
    int ki;
    fm_reduce<CB>(y, k, r, ki);
    const double p = fm_expm1_poly<CB>(r);
    const double s = fm_pow2i(ki);
    return fma(s, p, s);
}

// a / b for b >= 1 (finite or +inf): rcp.approx, one Newton step (~2x the
// seed's bits), then the residual correction q + (a - b q) y, whose error is
// the product of q's and y's (tests/test_fastmath_gpu.py: 0 ulp vs a / b)
__device__ __forceinline__ double fm_rcp(double b) {
    double y;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(b));
    const double e = fma(-b, y, 1.0);
    return fma(y, e, y);
}
// the quotient given y = fm_rcp(b) (shared by several quotients of one b)
__device__ __forceinline__ double fm_div_y(double a, double b, double y) {
    const double q = a * y;
    const double rr = fma(-b, q, a);
    return fma(rr, y, q);
}
__device__ __forceinline__ double fm_div(double a, double b) { return fm_div_y(a, b, fm_rcp(b)); }

// LSTM gate activation without branches: sigmoid(x) = 1 / (2 + expm1(-x)),
// tanh(x) = sign(x) (-e) / (2 + e) with e = expm1(-2|x|)
template <bool CB = false>
__device__ __forceinline__ double fm_gate_act(double x, bool is_tanh) {
    const double e = fm_expm1<CB>(is_tanh ? -2.0 * fabs(x) : -x);
    const double r = fm_div(is_tanh ? -e : 1.0, 2.0 + e);
    return is_tanh ? copysign(r, x) : r;
}

}  // namespace dp
