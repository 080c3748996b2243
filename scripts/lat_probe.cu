// Dependent-chain latency probe for the fp64 operations the policy kernels use.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o lat_probe lat_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

#define N 1024

__global__ void probe(double *out, long long *cyc, double a) {
    double x = a + threadIdx.x * 1e-9;
    long long t0, t1;
    // DFMA chain
    t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < N; i++) x = fma(x, 0.9999999, 1e-9);
    t1 = clock64();
    cyc[0] = t1 - t0;
    // DADD chain
    t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < N; i++) x = x + 1e-9;
    t1 = clock64();
    cyc[1] = t1 - t0;
    // exp chain
    t0 = clock64();
    for (int i = 0; i < N / 16; i++) x = exp(-x) + 0.5;
    t1 = clock64();
    cyc[2] = (t1 - t0) * 16;
    // tanh chain
    t0 = clock64();
    for (int i = 0; i < N / 16; i++) x = tanh(x) + 0.5;
    t1 = clock64();
    cyc[3] = (t1 - t0) * 16;
    // div chain
    t0 = clock64();
    for (int i = 0; i < N / 16; i++) x = 1.0 / (1.0 + x);
    t1 = clock64();
    cyc[4] = (t1 - t0) * 16;
    // log chain
    t0 = clock64();
    for (int i = 0; i < N / 16; i++) x = log(x + 2.0);
    t1 = clock64();
    cyc[5] = (t1 - t0) * 16;
    // shfl chain
    t0 = clock64();
    for (int i = 0; i < N / 16; i++) x = __shfl_xor_sync(0xffffffffu, x, 1) + 1e-9;
    t1 = clock64();
    cyc[6] = (t1 - t0) * 16;
    out[threadIdx.x] = x;
}

__global__ void probe_smem(double *out, long long *cyc) {
    __shared__ double s[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) s[i] = (i * 7 + 1) % 1024;
    __syncthreads();
    int idx = 0;
    double x = 0;
    long long t0 = clock64();
    for (int i = 0; i < N; i++) {
        x = s[idx];
        idx = (int)x;
    }
    long long t1 = clock64();
    cyc[7] = t1 - t0;
    long long t2 = clock64();
    for (int i = 0; i < 256; i++) __syncthreads();
    long long t3 = clock64();
    cyc[8] = (t3 - t2) * 4;
    out[threadIdx.x] = x;
}

int main() {
    double *out;
    long long *cyc, h[16];
    cudaMalloc(&out, 1024 * 8);
    cudaMalloc(&cyc, 16 * 8);
    for (int rep = 0; rep < 2; rep++) {
        probe<<<1, 32>>>(out, cyc, 0.3);
        probe_smem<<<1, 256>>>(out, cyc);
        cudaDeviceSynchronize();
    }
    cudaMemcpy(h, cyc, 16 * 8, cudaMemcpyDeviceToHost);
    const char *names[] = {"dfma", "dadd", "exp+add", "tanh+add", "div(1/(1+x))", "log(x+2)", "shfl+add",
                           "lds chain", "syncthreads(256thr)"};
    for (int i = 0; i < 9; i++) printf("%-22s %8.1f cycles/op\n", names[i], (double)h[i] / N);
    return 0;
}
