// Latency of LSTM gate-activation variants for one warp whose lanes mix the
// 3 sigmoid gates and the tanh gate (lane & 3 == 3), as in the policy kernels.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -o act_probe act_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ double act_ref(double x, bool t) { return t ? tanh(x) : 1.0 / (1.0 + exp(-x)); }
__device__ __forceinline__ double act_expm1(double x, bool t) {
    const double e = expm1(t ? -2.0 * fabs(x) : -x);
    const double r = (t ? -e : 1.0) / (2.0 + e);
    return t ? copysign(r, x) : r;
}
__device__ __forceinline__ double act_exp(double x, bool t) {  // tanh via exp (abs-accurate)
    const double e = exp(t ? -2.0 * fabs(x) : -x);
    const double r = (t ? 1.0 - e : 1.0) / (1.0 + e);
    return t ? copysign(r, x) : r;
}

template <int V>
__global__ void probe(double *out, long long *cyc) {
    const bool t = (threadIdx.x & 3) == 3;
    double x = 0.1 + threadIdx.x * 1e-3;
    long long t0 = clock64();
    for (int i = 0; i < 256; i++) {
        const double y = V == 0 ? act_ref(x, t) : V == 1 ? act_expm1(x, t) : act_exp(x, t);
        x = y * 0.5 + 0.1;
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[V] = (t1 - t0) / 256;
    out[threadIdx.x] = x;
}

int main() {
    double *out;
    long long *cyc, h[4];
    cudaMalloc(&out, 1024 * 8);
    cudaMalloc(&cyc, 8 * 8);
    for (int rep = 0; rep < 2; rep++) {
        probe<0><<<1, 32>>>(out, cyc);
        probe<1><<<1, 32>>>(out, cyc);
        probe<2><<<1, 32>>>(out, cyc);
        cudaDeviceSynchronize();
    }
    cudaMemcpy(h, cyc, 32, cudaMemcpyDeviceToHost);
    printf("ref (tanh | 1/(1+exp))  %lld cycles/act\nexpm1 unified            %lld cycles/act\nexp unified              %lld cycles/act\n",
           h[0], h[1], h[2]);
    return 0;
}
