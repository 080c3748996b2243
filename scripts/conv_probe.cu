// Throughput probe: fp64 -> 6 balanced int8 digit planes (tc.cuh digits6) on
// one SM, 16 warps, three conversion variants.  Prints cycles per element.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_1706_04972_b200/csrc scripts/conv_probe.cu -o /tmp/conv_probe
#include <cstdio>
#include <cstdint>

#include "tc.cuh"

template <int V>
__device__ __forceinline__ unsigned long long conv(double x, double s) {
    if (V == 0) return dp::tc::digits6(x, s);  // DFMA magic
    if (V == 1) {                               // DMUL + F2I
        const long long v = __double2ll_rn(x * s);
        return ((unsigned long long)v + dp::tc::kBias) ^ dp::tc::kBias;
    }
    // integer-only: shift the mantissa (s folded into a per-column shift)
    const unsigned long long b = (unsigned long long)__double_as_longlong(x);
    const int e = (int)((b >> 52) & 0x7FF);
    const unsigned long long m = (b & 0xFFFFFFFFFFFFFull) | (e ? 0x10000000000000ull : 0ull);
    const int sh = 1075 - (int)s - e;  // s carries the shift exponent here
    unsigned long long v = sh >= 64 ? 0ull : (sh > 0 ? m >> sh : m << -sh);
    v = (b >> 63) ? (0ull - v) : v;
    return (v + dp::tc::kBias) ^ dp::tc::kBias;
}

template <int V>
__global__ void __launch_bounds__(512) probe(const double *src, uint32_t *out, long long *cyc, int iters) {
    __shared__ __align__(16) double tile[32 * 128];
    __shared__ uint32_t planes[4096];
    for (int i = threadIdx.x; i < 32 * 128; i += blockDim.x) tile[i] = src[i];
    __syncthreads();
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const double s0 = V == 2 ? 1040.0 : 1099511627776.0;
    long long t0 = clock64();
    uint32_t acc = 0;
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int j = 0; j < 2; j++) {
            const int k = w + 16 * j;
            const double2 a = *reinterpret_cast<const double2 *>(tile + k * 128 + lane * 4);
            const double2 b = *reinterpret_cast<const double2 *>(tile + k * 128 + lane * 4 + 2);
            const unsigned long long u0 = conv<V>(a.x, s0), u1 = conv<V>(a.y, s0), u2 = conv<V>(b.x, s0),
                                     u3 = conv<V>(b.y, s0);
            const uint32_t x = __byte_perm((uint32_t)u0, (uint32_t)u1, 0x5140) ^ __byte_perm((uint32_t)u2, (uint32_t)u3, 0x7362) ^
                               (uint32_t)(u0 >> 32) ^ (uint32_t)(u3 >> 32);
            planes[(k * 32 + lane + it) & 4095] = x;
            acc ^= x;
        }
        __syncthreads();
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
    out[threadIdx.x] = acc + planes[threadIdx.x];
}

int main() {
    double *src;
    uint32_t *out;
    long long *cyc, h;
    cudaMalloc(&src, 32 * 128 * 8);
    cudaMalloc(&out, 512 * 4);
    cudaMalloc(&cyc, 8);
    double hs[32 * 128];
    for (int i = 0; i < 32 * 128; i++) hs[i] = (i % 7 - 3) * 0.123456789 + i * 1e-3;
    cudaMemcpy(src, hs, sizeof hs, cudaMemcpyHostToDevice);
    const int iters = 1000;
    const double elems = 32.0 * 128 * iters;
    probe<0><<<1, 512>>>(src, out, cyc, iters);
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("DFMA magic : %.3f cycles/element (%.0f cycles per 32x128 step)\n", h / elems, h / (double)iters);
    probe<1><<<1, 512>>>(src, out, cyc, iters);
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("DMUL + F2I : %.3f cycles/element (%.0f cycles per step)\n", h / elems, h / (double)iters);
    probe<2><<<1, 512>>>(src, out, cyc, iters);
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("int shifts : %.3f cycles/element (%.0f cycles per step)\n", h / elems, h / (double)iters);
    return 0;
}
