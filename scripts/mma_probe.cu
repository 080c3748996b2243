// Issue-rate probe for tcgen05.mma kind::i8 on one SM: cycles per MMA for
// M=128, N in {80, 128, 256}, K-major vs MN-major operands (no swizzle).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_1706_04972_b200/csrc scripts/mma_probe.cu -o scripts/_mma_probe
#include <cstdio>
#include <cstdint>

#include "tc.cuh"

using namespace dp::tc;

__host__ __device__ constexpr uint32_t idesc_i8(int M, int N, int amaj, int bmaj) {
    return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)amaj << 15) | ((uint32_t)bmaj << 16) |
           ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__global__ void probe(int N, int mn, int n_mma, long long *out) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tm;
    for (int i = threadIdx.x; i < 64 * 1024; i += blockDim.x) sm[i] = (uint8_t)(i * 7);
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        fence_mbar_init();
    }
    if (threadIdx.x < 32) tmem_alloc(&tm, 512);
    fence_async_smem();
    fence_before();
    __syncthreads();
    fence_after();
    if (threadIdx.x == 0) {
        const uint32_t a = smem_u32(sm), b = a + 32 * 1024;
        // K-major: core (8 rows x 16 B) at [grp][khalf]: LBO = 128 (k), SBO = 256 (rows)
        // MN-major: core (16 B of MN x 8 k rows): SBO = 128 (MN groups), LBO = (M/16)*128 (k groups)
        const uint64_t ad = mn ? smem_desc(a, 8 * 128, 128) : smem_desc(a, 128, 256);
        const uint64_t bd = mn ? smem_desc(b, (N / 16) * 128, 128) : smem_desc(b, 128, 256);
        const uint32_t id = idesc_i8(128, N, mn, mn);
        const int cols = N <= 80 ? 80 : N;  // accumulator stride
        const int nacc = 512 / cols;
        long long t0 = clock64();
        for (int i = 0; i < n_mma; i++) mma_i8(tm + (i % nacc) * cols, ad, bd, id, 1u);
        mma_commit(&bar);
        mbar_wait(&bar, 0);
        long long t1 = clock64();
        out[0] = t1 - t0;
    }
    __syncthreads();
    if (threadIdx.x < 32) tmem_dealloc(tm, 512);
}

int main() {
    long long *d, h;
    cudaMalloc(&d, 8);
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    const int n = 4200;
    for (int mn = 0; mn < 2; mn++)
        for (int N : {80, 128, 256}) {
            probe<<<1, 128, 64 * 1024>>>(N, mn, n, d);
            cudaError_t e = cudaDeviceSynchronize();
            cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
            const double macs = 128.0 * N * 32;
            printf("%s N=%3d: %.1f cycles/MMA  (%.0f int8 MAC/clk)  %s\n", mn ? "MN-major" : "K-major ", N,
                   h / (double)n, macs * n / h, e == cudaSuccess ? "" : cudaGetErrorString(e));
        }
    return 0;
}
