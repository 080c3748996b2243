// Probe: tcgen05.mma kind::i8 with the A operand in TMEM (M=128, K=32 per MMA),
// small N (16): correctness vs the same MMA with A from shared memory, issue
// rate, and the latency of a 12-MMA batch (issue -> commit -> mbarrier).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_1706_04972_b200/csrc scripts/tmem_a_probe.cu -o scripts/_tmem_a_probe
#include <cstdio>
#include <cstdint>

#include "tc.cuh"

using namespace dp::tc;

__host__ __device__ constexpr uint32_t idesc_k(int M, int N) {  // s8 x s8 -> s32, both K-major
    return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void mma_i8_ta(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc,
                                          uint32_t acc) {
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d_tmem),
        "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(acc)
        : "memory");
}
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t (&v)[8]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"r"(taddr),
                 "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
                 : "memory");
}
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

__global__ void probe(const int8_t *A, const int8_t *B, int *out_s, int *out_t, long long *cyc) {
    __shared__ __align__(1024) int8_t sa[128 * 32];
    __shared__ __align__(1024) int8_t sb[16 * 32];
    __shared__ uint64_t bar;
    __shared__ uint32_t tm;
    const int tid = threadIdx.x;
    // K-major no-swizzle canonical layout: core (8 rows x 16 B) at [row/8][k/16]: SBO = 256, LBO = 128
    for (int x = tid; x < 128 * 32; x += blockDim.x) {
        const int m = x / 32, k = x % 32;
        sa[(m / 8) * 256 + (k / 16) * 128 + (m % 8) * 16 + (k % 16)] = A[x];
    }
    for (int x = tid; x < 16 * 32; x += blockDim.x) {
        const int n = x / 32, k = x % 32;
        sb[(n / 8) * 256 + (k / 16) * 128 + (n % 8) * 16 + (k % 16)] = B[x];
    }
    if (tid == 0) {
        mbar_init(&bar, 1);
        fence_mbar_init();
    }
    if (tid < 32) tmem_alloc(&tm, 256);
    fence_async_smem();
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t T = tm;
    // A into TMEM columns [64, 72): lane m holds row m's 32 bytes (k = 4c + byte)
    {
        const int m = tid;  // 128 threads = 4 warps = 128 lanes
        uint32_t v[8];
        for (int c = 0; c < 8; c++) {
            uint32_t w = 0;
            for (int b = 0; b < 4; b++) w |= (uint32_t)(uint8_t)A[m * 32 + 4 * c + b] << (8 * b);
            v[c] = w;
        }
        tmem_st8(T + ((uint32_t)((tid >> 5) * 32) << 16) + 64, v);
        tmem_st_wait();
    }
    fence_before();
    __syncthreads();
    fence_after();
    const uint64_t ad = smem_desc(smem_u32(sa), 128, 256), bd = smem_desc(smem_u32(sb), 128, 256);
    const uint32_t id = idesc_k(128, 16);
    uint32_t ph = 0;
    if (tid == 0) {
        mma_i8(T + 0, ad, bd, id, 0u);         // D0 = A(smem) B
        mma_i8_ta(T + 16, T + 64, bd, id, 0u);  // D1 = A(tmem) B
        mma_commit(&bar);
    }
    mbar_wait(&bar, ph);
    ph ^= 1;
    fence_after();
    {
        uint32_t v0[8], v1[8], w0[8], w1[8];
        const uint32_t base = T + ((uint32_t)((tid >> 5) * 32) << 16);
        tmem_ld8(base + 0, v0);
        tmem_ld8(base + 8, v1);
        tmem_ld8(base + 16, w0);
        tmem_ld8(base + 24, w1);
        tmem_ld_wait();
        for (int j = 0; j < 8; j++) {
            out_s[tid * 16 + j] = (int)v0[j];
            out_s[tid * 16 + 8 + j] = (int)v1[j];
            out_t[tid * 16 + j] = (int)w0[j];
            out_t[tid * 16 + 8 + j] = (int)w1[j];
        }
    }
    __syncthreads();
    // issue rate: 1200 MMAs with A in TMEM
    if (tid == 0) {
        long long t0 = clock64();
        for (int i = 0; i < 1200; i++) mma_i8_ta(T + (i % 8) * 16, T + 64, bd, id, 1u);
        mma_commit(&bar);
        mbar_wait(&bar, ph);
        cyc[0] = clock64() - t0;
        ph ^= 1;
        // same with A from shared memory
        t0 = clock64();
        for (int i = 0; i < 1200; i++) mma_i8(T + (i % 8) * 16, ad, bd, id, 1u);
        mma_commit(&bar);
        mbar_wait(&bar, ph);
        cyc[1] = clock64() - t0;
        ph ^= 1;
        // latency of a 12-MMA batch (x100)
        t0 = clock64();
        for (int r = 0; r < 100; r++) {
            for (int i = 0; i < 12; i++) mma_i8_ta(T + (i % 6) * 16, T + 64, bd, id, 1u);
            mma_commit(&bar);
            mbar_wait(&bar, ph);
            ph ^= 1;
        }
        cyc[2] = clock64() - t0;
        // latency of 1 MMA (x100)
        t0 = clock64();
        for (int r = 0; r < 100; r++) {
            mma_i8_ta(T, T + 64, bd, id, 1u);
            mma_commit(&bar);
            mbar_wait(&bar, ph);
            ph ^= 1;
        }
        cyc[3] = clock64() - t0;
    }
    fence_before();
    __syncthreads();
    if (tid < 32) {
        fence_after();
        tmem_dealloc(T, 256);
    }
}

int main() {
    int8_t hA[128 * 32], hB[16 * 32];
    for (int i = 0; i < 128 * 32; i++) hA[i] = (int8_t)((i * 37 + 11) % 255 - 127);
    for (int i = 0; i < 16 * 32; i++) hB[i] = (int8_t)((i * 53 + 7) % 255 - 127);
    int ref[128 * 16];
    for (int m = 0; m < 128; m++)
        for (int n = 0; n < 16; n++) {
            int s = 0;
            for (int k = 0; k < 32; k++) s += hA[m * 32 + k] * hB[n * 32 + k];
            ref[m * 16 + n] = s;
        }
    int8_t *dA, *dB;
    int *os, *ot;
    long long *cyc, hc[4];
    cudaMalloc(&dA, sizeof hA);
    cudaMalloc(&dB, sizeof hB);
    cudaMalloc(&os, 4 * 128 * 16);
    cudaMalloc(&ot, 4 * 128 * 16);
    cudaMalloc(&cyc, 32);
    cudaMemcpy(dA, hA, sizeof hA, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, hB, sizeof hB, cudaMemcpyHostToDevice);
    probe<<<1, 128>>>(dA, dB, os, ot, cyc);
    cudaError_t e = cudaDeviceSynchronize();
    int hs[128 * 16], ht[128 * 16];
    cudaMemcpy(hs, os, sizeof hs, cudaMemcpyDeviceToHost);
    cudaMemcpy(ht, ot, sizeof ht, cudaMemcpyDeviceToHost);
    cudaMemcpy(hc, cyc, sizeof hc, cudaMemcpyDeviceToHost);
    int bad_s = 0, bad_t = 0;
    for (int i = 0; i < 128 * 16; i++) {
        bad_s += hs[i] != ref[i];
        bad_t += ht[i] != ref[i];
    }
    printf("status %s; smem-A mismatches %d, tmem-A mismatches %d (of 2048)\n", cudaGetErrorString(e), bad_s, bad_t);
    printf("A in TMEM  : %.1f cycles/MMA (M128 N16 K32)\n", hc[0] / 1200.0);
    printf("A in smem  : %.1f cycles/MMA\n", hc[1] / 1200.0);
    printf("12-MMA batch + commit + wait: %.0f cycles\n", hc[2] / 100.0);
    printf("1 MMA + commit + wait       : %.0f cycles\n", hc[3] / 100.0);
    return 0;
}
