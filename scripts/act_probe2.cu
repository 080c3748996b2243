// Throughput/latency of the decoder's A-phase activation work: 256 threads
// (8 warps, one CTA), each evaluating gate_act for 2 independent samples per
// step (as dec_kernel<2> does), 256 dependent steps.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -o act_probe2 act_probe2.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ double gate_act(double x, bool t) {
    const double e = expm1(t ? -2.0 * fabs(x) : -x);
    const double r = (t ? -e : 1.0) / (2.0 + e);
    return t ? copysign(r, x) : r;
}

template <int NS, int THREADS>
__global__ void probe(double *out, long long *cyc) {
    const bool t = (threadIdx.x & 3) == 3;
    double x[NS];
    for (int m = 0; m < NS; m++) x[m] = 0.1 + threadIdx.x * 1e-3 + m * 0.01;
    __syncthreads();
    long long t0 = clock64();
    for (int i = 0; i < 256; i++) {
#pragma unroll
        for (int m = 0; m < NS; m++) x[m] = gate_act(x[m], t) * 0.5 + 0.1;
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[0] = (t1 - t0) / 256;
    double s = 0;
    for (int m = 0; m < NS; m++) s += x[m];
    out[threadIdx.x] = s;
}

int main() {
    double *out;
    long long *cyc, h;
    cudaMalloc(&out, 4096 * 8);
    cudaMalloc(&cyc, 8 * 8);
    auto run = [&](auto kern, int threads, const char *name) {
        for (int rep = 0; rep < 2; rep++) kern<<<1, threads>>>(out, cyc);
        cudaDeviceSynchronize();
        cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
        printf("%-28s %lld cycles/step\n", name, h);
    };
    run(probe<1, 32>, 32, "1 warp, 1 sample");
    run(probe<2, 32>, 32, "1 warp, 2 samples");
    run(probe<1, 256>, 256, "8 warps, 1 sample");
    run(probe<2, 256>, 256, "8 warps, 2 samples");
    run(probe<4, 256>, 256, "8 warps, 4 samples");
    run(probe<2, 512>, 512, "16 warps, 2 samples");
    return 0;
}
