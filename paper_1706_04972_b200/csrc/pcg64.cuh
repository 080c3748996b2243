// numpy PCG64 (XSL-RR 128/64) on the device: jump-ahead + next double.
//
// Reproduces Generator.random() bit-exactly (numpy is the reference's RNG,
// pkg/policy.py:321 via default_rng streams, pkg/trainer.py:260-262): state
// s <- s*M + inc mod 2^128; output rotr64(hi^lo, s>>122) of the new state;
// double = (out >> 11) * 2^-53.  Draw n reads the state after n+1 steps.
#pragma once
#include <stdint.h>

namespace dp {

struct u128 {
    uint64_t hi, lo;
};

__host__ __device__ __forceinline__ u128 mul128(u128 a, u128 b) {
    u128 r;
    r.lo = a.lo * b.lo;
#ifdef __CUDA_ARCH__
    r.hi = __umul64hi(a.lo, b.lo) + a.lo * b.hi + a.hi * b.lo;
#else
    r.hi = (uint64_t)(((unsigned __int128)a.lo * b.lo) >> 64) + a.lo * b.hi + a.hi * b.lo;
#endif
    return r;
}

__host__ __device__ __forceinline__ u128 add128(u128 a, u128 b) {
    u128 r;
    r.lo = a.lo + b.lo;
    r.hi = a.hi + b.hi + (r.lo < a.lo ? 1ull : 0ull);
    return r;
}

constexpr uint64_t kPcgMulHi = 0x2360ED051FC65DA4ull;
constexpr uint64_t kPcgMulLo = 0x4385DF649FCCF645ull;

__host__ __device__ __forceinline__ u128 pcg_step(u128 s, u128 inc) {
    return add128(mul128(s, u128{kPcgMulHi, kPcgMulLo}), inc);
}

// state after n steps (square-and-multiply over the affine map)
__host__ __device__ inline u128 pcg_jump(u128 s, u128 inc, uint64_t n) {
    u128 am{0, 1}, ap{0, 0}, cm{kPcgMulHi, kPcgMulLo}, cp = inc;
    while (n) {
        if (n & 1) {
            am = mul128(am, cm);
            ap = add128(mul128(ap, cm), cp);
        }
        cp = mul128(add128(cm, u128{0, 1}), cp);
        cm = mul128(cm, cm);
        n >>= 1;
    }
    return add128(mul128(am, s), ap);
}

__host__ __device__ __forceinline__ double pcg_double(u128 s) {
    const uint64_t x = s.hi ^ s.lo;
    const unsigned rot = (unsigned)(s.hi >> 58);
    const uint64_t out = (x >> rot) | (x << ((64u - rot) & 63u));
    return (double)(out >> 11) * (1.0 / 9007199254740992.0);
}

}  // namespace dp
