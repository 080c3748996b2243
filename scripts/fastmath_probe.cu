// ulp error of fastmath.cuh against libm, and the 2-sample latency of the activation.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -I paper_1706_04972_b200/csrc -o fm fastmath_probe.cu
#include <cstdio>
#include <cuda_runtime.h>
#include "fastmath.cuh"
using namespace dp;

__device__ __forceinline__ double ref_act(double x, bool t) {
    const double e = expm1(t ? -2.0 * fabs(x) : -x);
    const double r = (t ? -e : 1.0) / (2.0 + e);
    return t ? copysign(r, x) : r;
}
__device__ long long ulps(double a, double b) {
    if (a == b) return 0;
    long long ia = __double_as_longlong(a), ib = __double_as_longlong(b);
    if ((ia < 0) != (ib < 0)) return 1LL << 62;
    long long d = ia - ib;
    return d < 0 ? -d : d;
}
__global__ void err_kernel(unsigned long long *mx) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    // x over [-60, 60] densely plus tails
    const double x = -60.0 + 120.0 * ((double)i / (double)(gridDim.x * (long long)blockDim.x));
    unsigned long long m0 = ulps(fm_gate_act(x, false), ref_act(x, false));
    unsigned long long m1 = ulps(fm_gate_act(x, true), ref_act(x, true));
    unsigned long long m2 = ulps(fm_exp(x * 10.0), exp(x * 10.0));
    unsigned long long m3 = ulps(fm_expm1(x * 0.01), expm1(x * 0.01));
    atomicMax(mx + 0, m0);
    atomicMax(mx + 1, m1);
    atomicMax(mx + 2, m2);
    atomicMax(mx + 3, m3);
}
template <int V>
__global__ void lat(double *out, long long *cyc) {
    const bool t = (threadIdx.x & 3) == 3;
    double x0 = 0.1 + threadIdx.x * 1e-3, x1 = 0.3 + threadIdx.x * 1e-3;
    long long t0 = clock64();
    for (int i = 0; i < 256; i++) {
        if (V == 0) { x0 = ref_act(x0, t) * 0.5 + 0.1; x1 = ref_act(x1, t) * 0.5 + 0.1; }
        else { x0 = fm_gate_act(x0, t) * 0.5 + 0.1; x1 = fm_gate_act(x1, t) * 0.5 + 0.1; }
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[V] = (t1 - t0) / 256;
    out[threadIdx.x] = x0 + x1;
}
int main() {
    unsigned long long *mx, h[4];
    cudaMalloc(&mx, 32);
    cudaMemset(mx, 0, 32);
    err_kernel<<<1 << 14, 256>>>(mx);
    cudaMemcpy(h, mx, 32, cudaMemcpyDeviceToHost);
    printf("max ulp: sigmoid %llu  tanh %llu  exp %llu  expm1 %llu\n", h[0], h[1], h[2], h[3]);
    double *out; long long *cyc, c[2];
    cudaMalloc(&out, 4096 * 8); cudaMalloc(&cyc, 16);
    for (int rep = 0; rep < 2; rep++) { lat<0><<<1, 256>>>(out, cyc); lat<1><<<1, 256>>>(out, cyc); }
    cudaDeviceSynchronize();
    cudaMemcpy(c, cyc, 16, cudaMemcpyDeviceToHost);
    printf("8 warps x 2 samples: libm %lld cycles/step, fastmath %lld cycles/step\n", c[0], c[1]);
    return 0;
}
