// Dependent-chain latencies (cycles per op, one warp) of the fp64 / shuffle /
// shared-memory operations on the decoder's draw chain.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../paper_1706_04972_b200/csrc -o _lat_probe2 lat_probe2.cu
#include <cstdio>
#include <cuda_runtime.h>
#include "fastmath.cuh"
using namespace dp;

#define N 512
__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                 : "+d"(d[0]), "+d"(d[1]) : "d"(a), "d"(b));
}
__global__ void probe(double *out, long long *cyc, double a, int *idx) {
    __shared__ double sh[1024];
    __shared__ int si[1024];
    for (int i = threadIdx.x; i < 1024; i += 32) { sh[i] = 0.5 + i * 1e-6; si[i] = idx[i]; }
    __syncwarp();
    double x = a + threadIdx.x * 1e-9;
    long long t0, t1;
    int c = 0;
#define CH(k, body, n)                  \
    t0 = clock64();                     \
    for (int i = 0; i < (n); i++) { body; } \
    t1 = clock64();                     \
    cyc[k] = (t1 - t0) * 1000 / (n);
#pragma unroll 1
    for (int rep = 0; rep < 2; rep++) {
        CH(0, x = fma(x, 0.9999999, 1e-9), N)
        CH(1, x = x + 1e-9, N)
        CH(2, x = x * 0.99999999, N)
        CH(3, x = __shfl_xor_sync(0xffffffffu, x, 1) + 0.0, N)
        CH(4, x = __shfl_sync(0xffffffffu, x, (threadIdx.x + 1) & 31), N)
        CH(5, c = si[c], N)
        CH(6, x = sh[__double2int_rz(x) & 1] + 0.5, N)
        CH(7, x = fm_exp(-x) + 0.5, N)
        CH(8, x = fm_div(1.0, x + 1.0) + 0.5, N)
        CH(9, x = fm_gate_act(x, false) + 0.25, N)
        CH(10, x = fm_gate_act(x, true) + 0.25, N)
        CH(11, x = fmax(x, 0.25) + 1e-9, N)
        CH(12, x = (double)(__double2int_rn(x * 3.0) & 3) + x * 1e-3, N)
        CH(13, x = exp(-x) + 0.5, N)
        CH(14, { double y; asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x)); x = y + 0.5; }, N)
        CH(15, x = (x <= 0.7 ? 1.0 : 0.0) + x * 0.5, N)
        { double d[2] = {x, x}; CH(16, dmma(d, 0.5, 0.25), N) x += d[0]; }
        { double d[8][2] = {}; t0 = clock64(); for (int i = 0; i < N; i++) {
#pragma unroll
            for (int q = 0; q < 8; q++) dmma(d[q], 0.5, 0.25); } t1 = clock64(); cyc[17] = (t1 - t0) * 1000 / (8 * N);
          for (int q = 0; q < 8; q++) x += d[q][0]; }
    }
    out[threadIdx.x] = x + c;
}

int main() {
    double *out; long long *cyc; int *idx;
    cudaMalloc(&out, 32 * 8); cudaMallocManaged(&cyc, 32 * 8); cudaMallocManaged(&idx, 1024 * 4);
    for (int i = 0; i < 1024; i++) idx[i] = (i * 7 + 3) & 1023;
    probe<<<1, 32>>>(out, cyc, 0.3, idx);
    cudaDeviceSynchronize();
    const char *nm[18] = {"DFMA", "DADD", "DMUL", "shfl.xor f64 + add", "shfl idx f64", "LDS.32 chase", "LDS.64 dep (+F2I +add)",
                          "fm_exp + add", "fm_div + add", "gate_act sigmoid + add", "gate_act tanh + add", "fmax + add",
                          "F2I/I2F + fma", "libm exp + add", "rcp.approx.f64 + add", "compare-select + fma",
                          "DMMA m8n8k4 dependent", "DMMA 8 independent (1 warp)"};
    for (int k = 0; k < 18; k++) printf("%-28s %8.1f cycles\n", nm[k], cyc[k] / 1000.0);
    return 0;
}
