// Probe: where does tcgen05.mma (kind::i8, cta_group::1) put the M=64 accumulator
// in TMEM?  D = A (64x32) B^T (16x32) with A from shared memory; every lane of
// the 4 warp quarters reads 16 columns and the host matches lanes to rows.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_1706_04972_b200/csrc scripts/tmem_m64_probe.cu -o scripts/_tmem_m64_probe
#include <cstdio>
#include <cstdint>

#include "tc.cuh"

using namespace dp::tc;

__host__ __device__ constexpr uint32_t idesc_k(int M, int N) {
    return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__global__ void probe(const int8_t *A, const int8_t *B, int *out) {
    __shared__ __align__(1024) int8_t sa[64 * 32];
    __shared__ __align__(1024) int8_t sb[16 * 32];
    __shared__ uint64_t bar;
    __shared__ uint32_t tm;
    const int tid = threadIdx.x;
    for (int x = tid; x < 64 * 32; x += blockDim.x) {
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
    if (tid < 32) tmem_alloc(&tm, 64);
    fence_async_smem();
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t T = tm;
    // zero the accumulator region first (tcgen05.st), then D = A B
    {
        uint32_t z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"r"(
                         T + ((uint32_t)((tid >> 5) * 32) << 16)),
                     "r"(z[0]), "r"(z[1]), "r"(z[2]), "r"(z[3]), "r"(z[4]), "r"(z[5]), "r"(z[6]), "r"(z[7])
                     : "memory");
        asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"r"(
                         T + 8 + ((uint32_t)((tid >> 5) * 32) << 16)),
                     "r"(z[0]), "r"(z[1]), "r"(z[2]), "r"(z[3]), "r"(z[4]), "r"(z[5]), "r"(z[6]), "r"(z[7])
                     : "memory");
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    fence_before();
    __syncthreads();
    fence_after();
    if (tid == 0) {
        mma_i8(T, smem_desc(smem_u32(sa), 128, 256), smem_desc(smem_u32(sb), 128, 256), idesc_k(64, 16), 0u);
        mma_commit(&bar);
    }
    mbar_wait(&bar, 0);
    fence_after();
    uint32_t v0[8], v1[8];
    const uint32_t base = T + ((uint32_t)((tid >> 5) * 32) << 16);
    tmem_ld8(base, v0);
    tmem_ld8(base + 8, v1);
    tmem_ld_wait();
    for (int j = 0; j < 8; j++) {
        out[tid * 16 + j] = (int)v0[j];
        out[tid * 16 + 8 + j] = (int)v1[j];
    }
    fence_before();
    __syncthreads();
    if (tid < 32) {
        fence_after();
        tmem_dealloc(T, 64);
    }
}

int main() {
    int8_t hA[64 * 32], hB[16 * 32];
    for (int i = 0; i < 64 * 32; i++) hA[i] = (int8_t)((i * 37 + 11) % 255 - 127);
    for (int i = 0; i < 16 * 32; i++) hB[i] = (int8_t)((i * 53 + 7) % 255 - 127);
    int ref[64 * 16];
    for (int m = 0; m < 64; m++)
        for (int n = 0; n < 16; n++) {
            int s = 0;
            for (int k = 0; k < 32; k++) s += hA[m * 32 + k] * hB[n * 32 + k];
            ref[m * 16 + n] = s;
        }
    int8_t *dA, *dB;
    int *o;
    cudaMalloc(&dA, sizeof hA);
    cudaMalloc(&dB, sizeof hB);
    cudaMalloc(&o, 4 * 128 * 16);
    cudaMemcpy(dA, hA, sizeof hA, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, hB, sizeof hB, cudaMemcpyHostToDevice);
    probe<<<1, 128>>>(dA, dB, o);
    cudaError_t e = cudaDeviceSynchronize();
    int h[128 * 16];
    cudaMemcpy(h, o, sizeof h, cudaMemcpyDeviceToHost);
    printf("status %s\n", cudaGetErrorString(e));
    // which row does each lane hold (columns 0..15 as a full row match)?
    for (int lane = 0; lane < 128; lane++) {
        int row = -1, partial = -1;
        for (int m = 0; m < 64; m++) {
            int match = 0;
            for (int n = 0; n < 16; n++) match += h[lane * 16 + n] == ref[m * 16 + n];
            if (match == 16) row = m;
            else if (match >= 4 && partial < 0) partial = m;
        }
        bool zero = true;
        for (int n = 0; n < 16; n++) zero &= h[lane * 16 + n] == 0;
        printf("lane %3d: %s%d%s\n", lane, row >= 0 ? "row " : (zero ? "zero " : "other (partial row "), row >= 0 ? row : partial,
               row >= 0 || zero ? "" : ")");
    }
    return 0;
}
