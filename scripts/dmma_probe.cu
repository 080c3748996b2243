// DMMA (mma.sync m8n8k4 f64) vs DFMA throughput probe on one GPU.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/dmma_probe scripts/dmma_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d[0]), "+d"(d[1]) : "d"(a), "d"(b));
}

template <int CH>
__global__ void dmma_kernel(int iters, double *out) {
    double acc[CH][2];
    for (int c = 0; c < CH; c++) acc[c][0] = acc[c][1] = 0.0;
    double a = threadIdx.x * 1e-3, b = 1.0 + blockIdx.x * 1e-6;
    for (int i = 0; i < iters; i++) {
#pragma unroll
        for (int c = 0; c < CH; c++) dmma(acc[c], a, b);
    }
    double s = 0;
    for (int c = 0; c < CH; c++) s += acc[c][0] + acc[c][1];
    if (s == 12345.0) out[0] = s;
}

__global__ void dfma_kernel(int iters, double *out) {
    double acc[8];
    for (int c = 0; c < 8; c++) acc[c] = c;
    double a = threadIdx.x * 1e-3, b = 1.0;
    for (int i = 0; i < iters; i++) {
#pragma unroll
        for (int c = 0; c < 8; c++) acc[c] = fma(a, acc[c], b);
    }
    double s = 0;
    for (int c = 0; c < 8; c++) s += acc[c];
    if (s == 12345.0) out[0] = s;
}

template <typename F>
float time_it(F f) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    f();
    cudaEventRecord(e0);
    f();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    return ms;
}

int main() {
    double *out;
    cudaMalloc(&out, 8);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int iters = 20000;
    for (int warps : {4, 8, 16}) {
        const int threads = 32 * warps;
        float ms = time_it([&] { dmma_kernel<8><<<sms, threads>>>(iters, out); });
        double flops = 2.0 * 256 * 8 * (double)iters * warps * sms;  // 256 FMA per warp-mma
        printf("DMMA  %2d warps/SM, 8 chains: %.2f TFLOP/s\n", warps, flops / ms / 1e9);
    }
    // latency: one warp per SM, CH independent chains
    {
        float ms1 = time_it([&] { dmma_kernel<1><<<sms, 32>>>(iters, out); });
        float ms2 = time_it([&] { dmma_kernel<2><<<sms, 32>>>(iters, out); });
        float ms4 = time_it([&] { dmma_kernel<4><<<sms, 32>>>(iters, out); });
        float ms8 = time_it([&] { dmma_kernel<8><<<sms, 32>>>(iters, out); });
        const double clk = 1.9e9;  // approximate SM clock for the cycle conversion
        printf("DMMA 1 warp/SM: cycles per mma with 1/2/4/8 chains: %.1f %.1f %.1f %.1f\n",
               ms1 * 1e-3 * clk / iters, ms2 * 1e-3 * clk / (2.0 * iters), ms4 * 1e-3 * clk / (4.0 * iters),
               ms8 * 1e-3 * clk / (8.0 * iters));
    }
    for (int warps : {8, 16, 32}) {
        const int threads = 32 * warps;
        float ms = time_it([&] { dfma_kernel<<<sms, threads>>>(iters, out); });
        double flops = 2.0 * 8 * (double)iters * threads * sms;
        printf("DFMA  %2d warps/SM, 8 chains: %.2f TFLOP/s\n", warps, flops / ms / 1e9);
    }
    return 0;
}
