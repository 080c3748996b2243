// Attention backward on the 5th-generation tensor cores (tcgen05 kind::i8
// digit planes, TMEM accumulators, TMA bulk copies): the GM / stored-numerator
// rows pass of the trainer's split backward (att_bwd_kernel<true, true>,
// policy_bwd.cu, is the fp64 DMMA version of the same arithmetic).
//
// Reference: grad_log_prob's attention terms (/root/reference/pkg/src/devplace/
// policy.py:378-395 with the forward of policy.py:294-300): per decode step t of
// sample k, alpha = softmax(proj h_t), dalpha = dctx . enc_i, ds = alpha (dalpha -
// alpha . dalpha); dh_t += ds proj (through s = proj h), and the encoder-side
// sums G_k = sum_t ds_t^T h_t (d_enc = G W_att, dW_att = G^T enc in the grads
// pass) and A_k = sum_t alpha_t^T du_t (the context path).
//
// Per CTA: whole samples; per (sample, 64-step tile, 64-position chunk):
//   1. DA on the fp64 tensor cores (DMMA, k = dd): dalpha = du encW^T; alpha =
//      e * esc from the decoder's stored numerators; ds = alpha (dalpha - w)
//   2. ds / alpha -> int8 digit planes (tc.cuh): ds row-scaled (A of dq), ds and
//      alpha column-scaled (A of G and A); the tile's H and du, and the
//      per-update proj chunk (TMA bulk copy of planes formed once per update by
//      proj_digits_kernel), are the B operands, digit planes stacked along N
//   3. M = 64 MMAs: dq = ds proj (dh_ext) and A = alpha^T du, then G = ds^T H;
//      each digit plane b of A multiplies the B window of planes 5 - b .. 5 in
//      one MMA (diagonals 5 .. 5 + b of the 6 int32 accumulators)
//   4. TMEM -> fp64 (scaled): dq accumulates over the chunks in registers and
//      is added to dh_ext; G / A go to per-tile partials with plain coalesced
//      stores (the grads pass's weighted reduction sums the tiles)

#include "policy.cuh"
#include "tc.cuh"

namespace dp {

namespace {

constexpr int kAtThreads = 256;
constexpr int kAtR = 64;                 // decode steps per tile (MMA M of dq, K of G / A)
constexpr int kAtC = 64;                 // positions per chunk (K of dq, M of G / A)
constexpr int kAtLd = 66;                // fp64 row stride of the ds / alpha staging
constexpr int kPl = 64 * 64;             // one 64 x 64 int8 digit plane
constexpr int kStackLbo = 24 * 128;      // B stacked along N: 6 planes x 64 = 24 groups of 16 -> K-group stride
constexpr int kStack = 8 * kStackLbo;    // 64-deep K: 24576 B
constexpr int kDuLbo = 6 * 128;          // du planes: 6 x 16 = 6 groups
constexpr int kDuStack = 8 * kDuLbo;     // 6144 B
constexpr int kTmemCols = 512;
constexpr int kColA = 384;               // TMEM columns of the A accumulators (6 diagonals x 16)
constexpr int kOpLd = 20;                // fp64 row stride of the DMMA operands (8 g x 4 t -> 2 wavefronts)

__host__ __device__ constexpr uint32_t idesc_i8(int M, int N, int a_mn, int b_mn) {
    return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)a_mn << 15) | ((uint32_t)b_mn << 16) |
           ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

struct AtcSmem {
    uint8_t proj[kStack];   // B of dq: proj chunk digits [i/8][N group][i%8][16] (bulk copy)
    uint8_t hb[kStack];     // B of G: the tile's H digits [r/8][N group][r%8][16]
    uint8_t dub[kDuStack];  // B of A: the tile's du digits
    uint8_t adq[6 * kPl];   // A of dq: ds row-scaled, K-major [r/8][i/16][r%8][i%16]
    uint8_t ade[6 * kPl];   // A of G: ds column-scaled, MN-major (same byte layout)
    uint8_t ada[6 * kPl];   // A of A: alpha column-scaled
    double ds[kAtR * kAtLd];
    double al[kAtR * kAtLd];
    double du[kAtR * kOpLd];   // the tile's du rows (columns >= dd zero; padded: conflict-free DMMA fragments)
    double encw[kAtC * kOpLd]; // the chunk's encW rows
    double w[kAtR];
    double s_row[kAtR], s_ci[kAtC], s_ai[kAtC], s_du[16];  // 2^s scales
    double pinv[kH];                                        // 2^-s of the proj columns
    uint64_t bar_mma, bar_proj;
    uint32_t tmem;
};

// byte offset of (row-of-K or M index a, 16-byte-run index b) in the 64 x 64
// plane layout [a/8][b/16][a%8][b%16] (K-major for dq, MN-major for G / A)
__device__ __forceinline__ int pl_off(int a, int b) { return (a >> 3) * 512 + (b >> 4) * 128 + (a & 7) * 16 + (b & 15); }

// 4 consecutive elements' digits -> one word per plane at planes + p * stride + off
__device__ __forceinline__ void put4(uint8_t *planes, int stride, int off, const unsigned long long (&u)[4]) {
    const uint32_t l0 = (uint32_t)u[0], l1 = (uint32_t)u[1], l2 = (uint32_t)u[2], l3 = (uint32_t)u[3];
    const uint32_t h0 = (uint32_t)(u[0] >> 32), h1 = (uint32_t)(u[1] >> 32), h2 = (uint32_t)(u[2] >> 32),
                   h3 = (uint32_t)(u[3] >> 32);
    const uint32_t a = __byte_perm(l0, l1, 0x5140), b = __byte_perm(l0, l1, 0x7362);
    const uint32_t c = __byte_perm(l2, l3, 0x5140), d = __byte_perm(l2, l3, 0x7362);
    const uint32_t e = __byte_perm(h0, h1, 0x5140), f = __byte_perm(h2, h3, 0x5140);
    *reinterpret_cast<uint32_t *>(planes + 0 * stride + off) = __byte_perm(a, c, 0x5410);
    *reinterpret_cast<uint32_t *>(planes + 1 * stride + off) = __byte_perm(a, c, 0x7632);
    *reinterpret_cast<uint32_t *>(planes + 2 * stride + off) = __byte_perm(b, d, 0x5410);
    *reinterpret_cast<uint32_t *>(planes + 3 * stride + off) = __byte_perm(b, d, 0x7632);
    *reinterpret_cast<uint32_t *>(planes + 4 * stride + off) = __byte_perm(e, f, 0x5410);
    *reinterpret_cast<uint32_t *>(planes + 5 * stride + off) = __byte_perm(e, f, 0x7632);
}

__device__ __forceinline__ int expo(double v) { return (__double2hiint(v) >> 20) & 0x7FF; }

__device__ __forceinline__ void dmma884(double (&d)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d[0]), "+d"(d[1])
                 : "d"(a), "d"(b));
}

// one M = 64 digit-plane product: A planes (stride kPl, K step ka bytes), B
// stacked planes (N group stride 128 per 16 columns; plane c at column nb * c;
// K step kb bytes), accumulators at TMEM column d0 (6 diagonals x nb)
__device__ __forceinline__ void digit_gemm(uint32_t tmem, uint32_t d0, uint32_t a0, int a_lbo, int a_sbo, int a_mn,
                                           int ka, uint32_t b0, int b_lbo, int nb, int kb, int ksteps) {
    for (int ks = 0; ks < ksteps; ks++)
#pragma unroll
        for (int b = tc::kDigits - 1; b >= 0; b--) {
            const int ntot = (b + 1) * nb;
            const int n1 = ntot <= 256 ? ntot : 256;
            const uint64_t ad = tc::smem_desc(a0 + b * kPl + ks * ka, a_lbo, a_sbo);
            const uint32_t bs = b0 + (tc::kDigits - 1 - b) * (nb / 16) * 128 + ks * kb;
            const uint32_t acc = (ks == 0 && b == tc::kDigits - 1) ? 0u : 1u;
            tc::mma_i8(tmem + d0, ad, tc::smem_desc(bs, b_lbo, 128), idesc_i8(64, n1, a_mn, 1), acc);
            if (n1 < ntot)
                tc::mma_i8(tmem + d0 + n1, ad, tc::smem_desc(bs + (n1 / 16) * 128, b_lbo, 128),
                           idesc_i8(64, ntot - n1, a_mn, 1), acc);
        }
}

// 8 accumulator columns of this lane's row, summed over the 6 diagonals:
// out[j] = sum_e acc_e[j] 256^(e + 5), with the diagonals combined exactly in
// two int64 halves (|acc| < 2^31: lo = sum_{e<4} acc_e 2^8e < 2^56, hi = acc_4
// + 2^8 acc_5 < 2^40) and one fp64 fma
__device__ __forceinline__ void drain8(uint32_t taddr, int stride_e, double (&out)[8]) {
    uint32_t v[6][8];
#pragma unroll
    for (int e = 0; e < tc::kDiags; e++) tc::tmem_ld8(taddr + e * stride_e, v[e]);
    tc::tmem_ld_wait();
#pragma unroll
    for (int j = 0; j < 8; j++) {
        const long long lo = (long long)(int)v[0][j] + ((long long)(int)v[1][j] << 8) +
                             ((long long)(int)v[2][j] << 16) + ((long long)(int)v[3][j] << 24);
        const long long hi = (long long)(int)v[4][j] + ((long long)(int)v[5][j] << 8);
        out[j] = fma((double)hi, tc::pow2(72), (double)lo * tc::pow2(40));
    }
}

__global__ void __launch_bounds__(kAtThreads, 1)
    att_bwd_tc_kernel(PolicyDims dm, int K, int samples_per_cta, const uint8_t *__restrict__ proj_dig,
                      const double *__restrict__ proj_inv, const double *__restrict__ encW,
                      const double *__restrict__ act_h, const double *__restrict__ row_w,
                      const double *__restrict__ row_du, const double *__restrict__ act_e,
                      const double *__restrict__ act_esc, double *__restrict__ tile_part,
                      double *__restrict__ tile_partA, double *__restrict__ row_dhx) {
    extern __shared__ uint8_t smem_raw[];
    AtcSmem &S = *reinterpret_cast<AtcSmem *>(smem_raw + ((128u - (tc::smem_u32(smem_raw) & 127u)) & 127u));
    const int tid = threadIdx.x, lane = tid & 31, wp = tid >> 5, g = lane >> 2, t4 = lane & 3;
    const int T = dm.T, dd = dm.dd;
    const int tps = (T + kAtR - 1) / kAtR, nch = (T + kAtC - 1) / kAtC;
    const int s_begin = blockIdx.x * samples_per_cta, s_end = min(K, s_begin + samples_per_cta);
    if (tid == 0) {
        tc::mbar_init(&S.bar_mma, 1);
        tc::mbar_init(&S.bar_proj, 1);
        tc::fence_mbar_init();
    }
    if (wp == 0) tc::tmem_alloc(&S.tmem, kTmemCols);
    if (tid < kH) S.pinv[tid] = proj_inv[tid];
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tmem = S.tmem;
    const uint32_t a_dq = tc::smem_u32(S.adq), a_de = tc::smem_u32(S.ade), a_da = tc::smem_u32(S.ada);
    const uint32_t b_proj = tc::smem_u32(S.proj), b_h = tc::smem_u32(S.hb), b_du = tc::smem_u32(S.dub);
    uint32_t ph_mma = 0, ph_proj = 0;
    // drain geometry (M = 64: row m lives in TMEM lane (m / 16) * 32 + m % 16):
    // warp w reads lanes 32 (w & 3) ..; its lanes 0-15 hold rows 16 (w & 3) + lane
    const int q = wp & 3, half = wp >> 2;
    const bool drow = lane < 16;
    const int dm_row = 16 * q + (lane & 15);
    const uint32_t tl_base = tmem + ((uint32_t)(q * 32) << 16);

    for (int smp = s_begin; smp < s_end; smp++) {
        for (int tl = 0; tl < tps; tl++) {
            const int t0 = tl * kAtR, nrow = min(kAtR, T - t0);
            const size_t rb = (size_t)smp * T + t0;
            // ---- tile operands: du, w (fp64) and the H / du digit planes
            for (int x = tid; x < kAtR * 16; x += kAtThreads) {
                const int r = x >> 4, o = x & 15;
                S.du[r * kOpLd + o] = (r < nrow && o < dd) ? row_du[(rb + r) * dd + o] : 0.0;
            }
            if (tid < kAtR) S.w[tid] = tid < nrow ? row_w[rb + tid] : 0.0;
            // H digits: |h| <= 1 -> fixed scale 2^45 (fix_shift of exponent 1023)
            for (int x = tid; x < kAtR * 16; x += kAtThreads) {
                const int r = x >> 4, j = (x & 15) * 4;
                unsigned long long u[4] = {0, 0, 0, 0};
                if (r < nrow) {
                    const double2 v01 = *reinterpret_cast<const double2 *>(act_h + (rb + r) * kH + j);
                    const double2 v23 = *reinterpret_cast<const double2 *>(act_h + (rb + r) * kH + j + 2);
                    const double sc = tc::pow2(45);
                    u[0] = tc::digits6(v01.x, sc);
                    u[1] = tc::digits6(v01.y, sc);
                    u[2] = tc::digits6(v23.x, sc);
                    u[3] = tc::digits6(v23.y, sc);
                }
                // plane p at N group 4p + j / 16
                put4(S.hb, 4 * 128, (r >> 3) * kStackLbo + (j >> 4) * 128 + (r & 7) * 16 + (j & 15), u);
            }
            __syncthreads();
            if (tid < 16) {
                int eb = 0;
                for (int r = 0; r < kAtR; r++) eb = max(eb, expo(S.du[r * kOpLd + tid]));
                S.s_du[tid] = tc::pow2(tc::fix_shift(eb));
            }
            __syncthreads();
            {
                // du digits: 64 rows x 16 columns, one 4-column word per thread
                const int r = tid >> 2, o = (tid & 3) * 4;
                unsigned long long u[4];
#pragma unroll
                for (int e = 0; e < 4; e++) u[e] = tc::digits6(S.du[r * kOpLd + o + e], S.s_du[o + e]);
                put4(S.dub, 128, (r >> 3) * kDuLbo + (r & 7) * 16 + o, u);
            }
            // encW rows of chunk 0 (later chunks are prefetched while the MMAs run)
            for (int x = tid; x < kAtC * 16; x += kAtThreads) {
                const int i = x >> 4, o = x & 15;
                S.encw[i * kOpLd + o] = (i < T && o < dd) ? encW[(size_t)i * dd + o] : 0.0;
            }
            double dq[32];  // dh_ext of (row dm_row, columns 32 half .. +32), over the chunks
#pragma unroll
            for (int j = 0; j < 32; j++) dq[j] = 0.0;
            for (int ch = 0; ch < nch; ch++) {
                const int i0 = ch * kAtC, ncol = min(kAtC, T - i0);
                // proj digit planes of the chunk: one TMA bulk copy (formed once per update)
                if (tid == 0) {
                    tc::mbar_expect_tx(&S.bar_proj, kStack);
                    tc::bulk_load(S.proj, proj_dig + (size_t)ch * kStack, kStack, &S.bar_proj);
                }
                // this lane's stored numerators (rows mr, columns n*8 + 2 t4 + e)
                const int mr = wp * 8 + g;
                const bool rok = mr < nrow;
                const size_t row = rb + (rok ? mr : 0);
                double ev[8][2];
#pragma unroll
                for (int n = 0; n < 8; n++)
#pragma unroll
                    for (int e = 0; e < 2; e++) {
                        const int i = n * 8 + 2 * t4 + e;
                        ev[n][e] = (rok && i < ncol) ? __ldg(act_e + row * T + i0 + i) : 0.0;
                    }
                const double esc0 = rok ? __ldg(act_esc + row * 8 + ((i0 & 255) >> 5)) : 0.0;
                const double esc1 = rok ? __ldg(act_esc + row * 8 + (((i0 + 32) & 255) >> 5)) : 0.0;
                __syncthreads();
                // ---- DA on DMMA: dalpha[mr, i] = du[mr] . encW[i] (k = 16, zero padded)
                double da[8][2];
#pragma unroll
                for (int n = 0; n < 8; n++) da[n][0] = da[n][1] = 0.0;
#pragma unroll
                for (int ks = 0; ks < 4; ks++) {
                    const double a = S.du[mr * kOpLd + ks * 4 + t4];
#pragma unroll
                    for (int n = 0; n < 8; n++) dmma884(da[n], a, S.encw[(n * 8 + g) * kOpLd + ks * 4 + t4]);
                }
                const double wv = S.w[mr];
#pragma unroll
                for (int n = 0; n < 8; n++)
#pragma unroll
                    for (int e = 0; e < 2; e++) {
                        const int i = n * 8 + 2 * t4 + e;
                        const double al = ev[n][e] * (n < 4 ? esc0 : esc1);
                        S.al[mr * kAtLd + i] = al;
                        S.ds[mr * kAtLd + i] = al * (da[n][e] - wv);
                    }
                __syncthreads();
                // ---- scales: ds row maxima (dq), ds / alpha column maxima (G / A)
                if (tid < 64) {
                    int eb = 0;
                    for (int i = 0; i < kAtC; i++) eb = max(eb, expo(S.ds[tid * kAtLd + i]));
                    S.s_row[tid] = tc::pow2(tc::fix_shift(eb));
                } else if (tid < 128) {
                    const int i = tid - 64;
                    int eb = 0;
                    for (int r = 0; r < kAtR; r++) eb = max(eb, expo(S.ds[r * kAtLd + i]));
                    S.s_ci[i] = tc::pow2(tc::fix_shift(eb));
                } else if (tid < 192) {
                    const int i = tid - 128;
                    int eb = 0;
                    for (int r = 0; r < kAtR; r++) eb = max(eb, expo(S.al[r * kAtLd + i]));
                    S.s_ai[i] = tc::pow2(tc::fix_shift(eb));
                }
                __syncthreads();
                // ---- digit planes: warp covers 8 rows x 16 columns per pass (conflict-free words)
#pragma unroll
                for (int pass = 0; pass < 4; pass++) {
                    const int G = wp + 8 * pass;       // 32 groups = 8 row octets x 4 column blocks
                    const int r = (G >> 2) * 8 + (lane >> 2), i = (G & 3) * 16 + (lane & 3) * 4;
                    const double *dsr = S.ds + r * kAtLd + i, *alr = S.al + r * kAtLd + i;
                    const double sr = S.s_row[r];
                    unsigned long long u[4], v[4], z[4];
#pragma unroll
                    for (int e = 0; e < 4; e++) {
                        u[e] = tc::digits6(dsr[e], sr);
                        v[e] = tc::digits6(dsr[e], S.s_ci[i + e]);
                        z[e] = tc::digits6(alr[e], S.s_ai[i + e]);
                    }
                    const int off = pl_off(r, i);
                    put4(S.adq, kPl, off, u);
                    put4(S.ade, kPl, off, v);
                    put4(S.ada, kPl, off, z);
                }
                tc::fence_async_smem();
                tc::mbar_wait(&S.bar_proj, ph_proj);
                ph_proj ^= 1;
                __syncthreads();
                // ---- dq = ds proj (M 64 rows, N 64 j, K 64 i) and A = alpha^T du (M 64 i, N 16, K 64 r)
                if (tid == 0) {
                    tc::fence_after();
                    digit_gemm(tmem, 0, a_dq, 128, 512, 0, 256, b_proj, kStackLbo, 64, 4 * kStackLbo, 2);
                    digit_gemm(tmem, kColA, a_da, 512, 128, 1, 2048, b_du, kDuLbo, 16, 4 * kDuLbo, 2);
                    tc::mma_commit(&S.bar_mma);
                }
                // the next chunk's encW rows: global loads in flight under the MMAs
                double enx[4];
                const bool more = ch + 1 < nch;
#pragma unroll
                for (int u = 0; u < 4; u++) {
                    const int x = tid + u * kAtThreads, i = (ch + 1) * kAtC + (x >> 4), o = x & 15;
                    enx[u] = (more && i < T && o < dd) ? __ldg(encW + (size_t)i * dd + o) : 0.0;
                }
                tc::mbar_wait(&S.bar_mma, ph_mma);
                ph_mma ^= 1;
                tc::fence_after();
                // staging of the drained G / A tiles (ds / alpha are consumed)
                double *stg = S.ds;  // [64][kAtLd]
#pragma unroll
                for (int c8 = 0; c8 < 32; c8 += 8) {
                    double v[8];
                    drain8(tl_base + half * 32 + c8, 64, v);
                    if (drow) {
                        const double ir = 1.0 / S.s_row[dm_row];
#pragma unroll
                        for (int j = 0; j < 8; j++) dq[c8 + j] += (v[j] * ir) * S.pinv[half * 32 + c8 + j];
                    }
                }
                {
                    double v[8];
                    drain8(tl_base + kColA + half * 8, 16, v);
                    if (drow) {
                        const double ii = 1.0 / S.s_ai[dm_row];
#pragma unroll
                        for (int j = 0; j < 8; j++) S.al[dm_row * kAtLd + half * 8 + j] = (v[j] * ii) / S.s_du[half * 8 + j];
                    }
                }
                tc::fence_before();
                __syncthreads();
                // ---- G = ds^T H (M 64 i, N 64 j, K 64 r)
                if (tid == 0) {
                    tc::fence_after();
                    digit_gemm(tmem, 0, a_de, 512, 128, 1, 2048, b_h, kStackLbo, 64, 4 * kStackLbo, 2);
                    tc::mma_commit(&S.bar_mma);
                }
                // the per-tile A partial (plain coalesced stores; the grads pass sums the tiles)
                {
                    double *pa = tile_partA + ((size_t)(smp * tps + tl) * T + i0) * dd;
                    for (int x = tid; x < ncol * dd; x += kAtThreads) {
                        const int i = x / dd, o = x - i * dd;
                        pa[x] = S.al[i * kAtLd + o];
                    }
                }
                tc::mbar_wait(&S.bar_mma, ph_mma);
                ph_mma ^= 1;
                tc::fence_after();
#pragma unroll
                for (int c8 = 0; c8 < 32; c8 += 8) {
                    double v[8];
                    drain8(tl_base + half * 32 + c8, 64, v);
                    if (drow) {
                        const double ii = tc::pow2(-45) / S.s_ci[dm_row];
#pragma unroll
                        for (int j = 0; j < 8; j++) stg[dm_row * kAtLd + half * 32 + c8 + j] = v[j] * ii;
                    }
                }
                tc::fence_before();
                __syncthreads();
                {
                    double *pe = tile_part + ((size_t)(smp * tps + tl) * T + i0) * kH;
                    for (int x = tid; x < ncol * kH; x += kAtThreads) pe[x] = stg[(x >> 6) * kAtLd + (x & 63)];
                }
                // encW rows of the next chunk (the DA of this chunk is long done)
                if (more)
#pragma unroll
                    for (int u = 0; u < 4; u++) {
                        const int x = tid + u * kAtThreads;
                        S.encw[(x >> 4) * kOpLd + (x & 15)] = enx[u];
                    }
                __syncthreads();  // the planes / staging of this chunk are rewritten next
            }
            // dh_ext += ds proj of the whole tile
            if (drow && dm_row < nrow) {
                double *dst = row_dhx + (rb + dm_row) * kH + half * 32;
#pragma unroll
                for (int j = 0; j < 32; j += 2) {
                    double2 *p2 = reinterpret_cast<double2 *>(dst + j);
                    const double2 o = *p2;
                    *p2 = make_double2(o.x + dq[j], o.y + dq[j + 1]);
                }
            }
        }
    }
    tc::fence_before();
    __syncthreads();
    if (wp == 0) {
        tc::fence_after();
        tc::tmem_dealloc(tmem, kTmemCols);
    }
}

// Per update: proj digit planes (B of dq) chunk by chunk in the shared-memory
// image the attention backward bulk-copies, column j scaled by its max over
// all T positions (proj_inv[j] = 2^-s_j).  One CTA.
__global__ void __launch_bounds__(256) proj_digits_kernel(int T, const double *__restrict__ proj,
                                                          uint8_t *__restrict__ out, double *__restrict__ proj_inv) {
    __shared__ int ebp[4][64];
    __shared__ double sc[64];
    const int tid = threadIdx.x, j = tid & 63, part = tid >> 6;
    int eb = 0;
    for (int i = part; i < T; i += 4) eb = max(eb, expo(proj[(size_t)i * kH + j]));
    ebp[part][j] = eb;
    __syncthreads();
    if (tid < 64) {
        const int e = max(max(ebp[0][tid], ebp[1][tid]), max(ebp[2][tid], ebp[3][tid]));
        const int s = tc::fix_shift(e);
        sc[tid] = tc::pow2(s);
        proj_inv[tid] = tc::pow2(-s);
    }
    __syncthreads();
    const int nch = (T + kAtC - 1) / kAtC;
    // element (i, j) of chunk c: planes stacked along N (plane p at N group 4p + j/16)
    for (int x = tid; x < nch * kAtC * 16; x += 256) {
        const int c = x / (kAtC * 16), rem = x - c * kAtC * 16, i = rem >> 4, jj = (rem & 15) * 4;
        const int ig = c * kAtC + i;
        unsigned long long u[4] = {0, 0, 0, 0};
        if (ig < T)
#pragma unroll
            for (int e = 0; e < 4; e++) u[e] = tc::digits6(proj[(size_t)ig * kH + jj + e], sc[jj + e]);
        put4(out + (size_t)c * kStack, 4 * 128, (i >> 3) * kStackLbo + (jj >> 4) * 128 + (i & 7) * 16 + (jj & 15), u);
    }
}

}  // namespace

size_t att_bwd_tc_smem() { return sizeof(AtcSmem) + 128; }
size_t att_bwd_tc_proj_bytes(int T) { return (size_t)((T + kAtC - 1) / kAtC) * kStack; }

bool att_bwd_tc_ok(const PolicyDims &dm) { return dm.dd <= 16; }

// the GM rows-pass attention backward on tcgen05: per-tile partials (G in
// tile_part, A in tile_partA; units = sample * tiles + tile), dh_ext += ds proj
// in row_dhx
int launch_att_bwd_tc(const PolicyDims &dm, int K, const double *proj, uint8_t *proj_dig, double *proj_inv,
                      const double *encW, const double *act_h, const double *row_w, const double *row_du,
                      const double *act_e, const double *act_esc, double *tile_part, double *tile_partA,
                      double *row_dhx, int n_cta, cudaStream_t st) {
    proj_digits_kernel<<<1, 256, 0, st>>>(dm.T, proj, proj_dig, proj_inv);
    DP_LAUNCH_CHECK();
    const int spc = ceil_div(K, n_cta);
    const size_t smem = att_bwd_tc_smem();
    DP_CUDA_TRY(cudaFuncSetAttribute(att_bwd_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    att_bwd_tc_kernel<<<ceil_div(K, spc), kAtThreads, smem, st>>>(dm, K, spc, proj_dig, proj_inv, encW, act_h, row_w,
                                                                 row_du, act_e, act_esc, tile_part, tile_partA, row_dhx);
    DP_LAUNCH_CHECK();
    return DP_OK;
}

}  // namespace dp
