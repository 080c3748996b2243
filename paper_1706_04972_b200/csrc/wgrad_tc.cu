// Decoder weight gradient on the 5th-generation tensor cores (tcgen05, TMEM,
// TMA), fp64-exact through int8 digit planes (tc.cuh).
//
// Reference: grad_log_prob's decoder weight terms (pkg/policy.py:378-395,
// gw_dec[dd:] += outer(h_prev, da), gw_dec[:dd] / gb_dec / dev_table via the
// input row) summed over samples by reinforce_update (pkg/trainer.py:138-154).
// Per CTA partial (same layout as dec_wgrad_kernel, policy_bwd.cu):
//   Hg[l][j]    = sum_r adv_r h_prev[r][l] da[r][j]        (l < 64)
//   DAsum[p][j] = sum_{r: prev choice p} adv_r da[r][j]    (p <= D)
// i.e. C^T with C[j][n] = sum_r da[r][j] Bm[r][n], Bm = [adv h_prev | adv onehot(prev)]:
// one GEMM with M = 128 gate columns per CTA (two CTAs per row chunk), N = 80
// (64 + D + 1 <= 80), contraction over the K*T rows (split-K over chunks).
//
// Roles (320 threads, one CTA per SM):
//   warp 0      TMA producer: fp64 tiles da[16 rows][128 cols] and
//               act_h[16 rows][64] (the previous rows' h) -> 5-slot ring
//   warp 1      MMA issuer (one thread): per 32-row step, the 21 digit-plane
//               pairs b + c >= 5 into 6 int32 TMEM accumulators (480 columns)
//   warps 2-9   converters: fp64 -> 6 int8 digit planes in the canonical
//               MN-major no-swizzle layout (row stride padded to 144 B so
//               every warp store is conflict-free); then the epilogue
//               (tcgen05.ld -> fp64) every <= 16K rows (int32 headroom) and
//               the partial store
// Column scales: da column j uses 2^s_j from the max exponent the decoder
// LSTM backward recorded (lstm_bwd_kernel colexp); Bm uses max|adv| (|h| < 1).

#include <cudaTypedefs.h>

#include "policy.cuh"
#include "tc.cuh"

namespace dp {

namespace {

constexpr int kWgM = 128;              // gate columns per CTA (MMA M)
constexpr int kWgN = 80;               // 64 h + (D+1) one-hot, padded to 16 (MMA N)
constexpr int kWgK = 32;               // rows per step (MMA K for int8)
constexpr int kWgSeg = 512;            // steps per TMEM drain: 6 * 2^14 * 16384 < 2^31 (debug mode 2: 3)
constexpr int kGrpStride = 144;        // bytes between 16-element MN groups (128 + 16 pad)
constexpr int kAPlane = (kWgK / 8) * (kWgM / 16) * kGrpStride;  // 4608
// B digit planes are stacked along N (plane c = rows [80 c, 80 c + 80) of a
// 480 x 32 operand), so one MMA multiplies A plane b with the window of B
// planes c = 5 - b .. 5 and writes the diagonals 5 .. 5 + b in one go (9 MMAs
// of N = 80..240 per step instead of 21 of N = 80: the MMA is bound by its
// shared-memory operand reads, ~91 cycles for any N <= 128 at K = 32,
// scripts/mma_probe.cu)
constexpr int kBPlane = (kWgN / 16) * kGrpStride;               // plane stride inside a k group (720)
constexpr int kALbo = (kWgM / 16) * kGrpStride;                 // k-group stride of A (1152)
constexpr int kBLbo = tc::kDigits * kBPlane;                    // k-group stride of B (4320)
constexpr int kI8Stage = tc::kDigits * kAPlane + (kWgK / 8) * kBLbo;  // 44928
// fp64 ring: slots of 16 rows (da 16 x 128 | h 16 x 64), 5 deep = 2.5 steps
// of TMA lookahead (~100 KB in flight per SM covers HBM latency)
constexpr int kSlotRows = 16, kSlots = 5;
constexpr int kDaSlot = kSlotRows * kWgM * 8, kHSlot = kSlotRows * kH * 8;
constexpr int kF64Slot = kDaSlot + kHSlot;                       // 24576
constexpr int kWgConv = 512;                                     // converter threads (warps 2-17)
constexpr int kConvWarps = kWgConv / 32;
constexpr int kEpCols = kWgN / (kConvWarps / 4);                 // epilogue columns per warp (20)
constexpr int kWgThreads = 64 + kWgConv;
constexpr int kTmemCols = 512;

struct WgBars {
    uint64_t f64_full[kSlots], f64_empty[kSlots], i8_full[2], i8_empty[2], acc_full, acc_empty;
    uint32_t tmem;
};
constexpr size_t kWgSmem =
    128 + (size_t)kSlots * kF64Slot + 2 * (size_t)kI8Stage + kWgM * sizeof(double) + sizeof(WgBars) + 64;

// byte offset of element (k, mn) inside a digit plane (MN-major, no swizzle):
// core matrix = 16 MN bytes x 8 k rows (16 B apart), MN groups kGrpStride
// apart, k groups lbo apart
__device__ __forceinline__ int plane_off(int k, int mn, int lbo) {
    return (k >> 3) * lbo + (mn >> 4) * kGrpStride + (k & 7) * 16 + (mn & 15);
}

// 4 consecutive MN elements (digits u[0..3]) -> one 32-bit word per plane
__device__ __forceinline__ void store_digits4(uint8_t *planes, int plane_bytes, int off,
                                              const unsigned long long (&u)[4]) {
    const uint32_t l0 = (uint32_t)u[0], l1 = (uint32_t)u[1], l2 = (uint32_t)u[2], l3 = (uint32_t)u[3];
    const uint32_t h0 = (uint32_t)(u[0] >> 32), h1 = (uint32_t)(u[1] >> 32), h2 = (uint32_t)(u[2] >> 32),
                   h3 = (uint32_t)(u[3] >> 32);
    const uint32_t a = __byte_perm(l0, l1, 0x5140), b = __byte_perm(l0, l1, 0x7362);
    const uint32_t c = __byte_perm(l2, l3, 0x5140), d = __byte_perm(l2, l3, 0x7362);
    const uint32_t e = __byte_perm(h0, h1, 0x5140), f = __byte_perm(h2, h3, 0x5140);
    uint32_t w[6];
    w[0] = __byte_perm(a, c, 0x5410);
    w[1] = __byte_perm(a, c, 0x7632);
    w[2] = __byte_perm(b, d, 0x5410);
    w[3] = __byte_perm(b, d, 0x7632);
    w[4] = __byte_perm(e, f, 0x5410);
    w[5] = __byte_perm(e, f, 0x7632);
#pragma unroll
    for (int p = 0; p < 6; p++) *reinterpret_cast<uint32_t *>(planes + p * plane_bytes + off) = w[p];
}

// (quotient, remainder) of a row index by T, advanced by 32 rows per step
struct RowPos {
    int q, r;
    __device__ __forceinline__ void init(int row, int T) { q = row / T, r = row - (row / T) * T; }
    __device__ __forceinline__ void advance(int T) {
        r += kWgK;
        while (r >= T) r -= T, q++;
    }
};

__global__ void __launch_bounds__(kWgThreads, 1)
    dec_wgrad_tc_kernel(const __grid_constant__ CUtensorMap map_da, const __grid_constant__ CUtensorMap map_h,
                        int T, int D, int rows, int steps_per_chunk, const double *__restrict__ enc_last,
                        const uint8_t *__restrict__ choice, const double *__restrict__ adv, int K,
                        const int *__restrict__ colexp, double *__restrict__ partial, size_t part_stride,
                        int seg_steps, int dbg /* timing ablations: 1 = no conversion, 2 = no TMA */) {
    extern __shared__ uint8_t smem_raw[];
    // 128-byte aligned base, kept as smem_raw + offset so every access stays a shared-window LDS/STS
    uint8_t *sm = smem_raw + ((128u - (tc::smem_u32(smem_raw) & 127u)) & 127u);
    uint8_t *f64s = sm;                              // [kSlots][da 16 x 128 | h 16 x 64]
    uint8_t *i8s = f64s + kSlots * kF64Slot;         // [2][6 A planes | 6 B planes]
    double *s_sa = reinterpret_cast<double *>(i8s + 2 * kI8Stage);  // [128] 2^s_j
    WgBars *bars = reinterpret_cast<WgBars *>(s_sa + kWgM);
    __shared__ double s_sb;
    __shared__ __align__(16) double s_enc[kH];
    __shared__ int s_eb[kWgConv / 32];

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int half = blockIdx.x & 1, chunk = blockIdx.x >> 1;
    const int n_steps_all = (rows + kWgK - 1) / kWgK;
    const int step0 = chunk * steps_per_chunk;
    const int nsteps = min(steps_per_chunk, n_steps_all - step0);
    if (nsteps <= 0) return;

    if (tid == 0) {
        for (int s = 0; s < kSlots; s++) {
            tc::mbar_init(&bars->f64_full[s], 1);
            tc::mbar_init(&bars->f64_empty[s], kWgConv / 32);
        }
        for (int s = 0; s < 2; s++) {
            tc::mbar_init(&bars->i8_full[s], kWgConv / 32);
            tc::mbar_init(&bars->i8_empty[s], 1);
        }
        tc::mbar_init(&bars->acc_full, 1);
        tc::mbar_init(&bars->acc_empty, kWgConv / 32);
        tc::fence_mbar_init();
        tc::tma_prefetch_desc(&map_da);
        tc::tma_prefetch_desc(&map_h);
    }
    if (warp == 0) tc::tmem_alloc(&bars->tmem, kTmemCols);
    if (tid >= 64) {
        const int c = tid - 64;
        // scales: A column (da) from its max exponent, B from max |adv|
        if (c < kWgM) s_sa[c] = tc::pow2(tc::fix_shift(colexp[half * kWgM + c]));
        int eb = adv ? 0 : 1023;
        if (adv)
            for (int k = c; k < K; k += kWgConv)
                eb = max(eb, (int)((unsigned long long)__double_as_longlong(adv[k]) >> 52) & 0x7FF);
        for (int o = 16; o; o >>= 1) eb = max(eb, __shfl_xor_sync(0xffffffffu, eb, o));
        if (lane == 0) s_eb[c >> 5] = eb;
        if (c < kH) s_enc[c] = enc_last[c];
    }
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    if (tid == 64) {
        int eb = 0;
        for (int w = 0; w < kConvWarps; w++) eb = max(eb, s_eb[w]);
        s_sb = tc::pow2(tc::fix_shift(eb));
    }
    __syncthreads();
    const uint32_t tmem = bars->tmem;

    if (warp == 0) {
        // ---------------- TMA producer: half-steps of 16 rows through the slot ring
        if (lane == 0) {
            const int nh = 2 * nsteps;
            for (int hs = 0; hs < nh; hs++) {
                const int s = hs % kSlots, use = hs / kSlots;
                if (use > 0) tc::mbar_wait(&bars->f64_empty[s], (use - 1) & 1);
                const int rb = step0 * kWgK + hs * kSlotRows;
                uint8_t *st = f64s + s * kF64Slot;
                if (dbg & 2) {
                    tc::mbar_arrive(&bars->f64_full[s]);
                    continue;
                }
                tc::mbar_expect_tx(&bars->f64_full[s], kF64Slot);
                tc::tma_load_2d(st, &map_da, &bars->f64_full[s], half * kWgM, rb);
                tc::tma_load_2d(st + kDaSlot, &map_h, &bars->f64_full[s], 0, rb - 1);
            }
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer
        if (lane == 0) {
            int seg = 0;
            for (int i = 0; i < nsteps; i++) {
                const int s = i & 1;
                const bool seg_first = i % seg_steps == 0;
                const bool seg_last = i % seg_steps == seg_steps - 1 || i == nsteps - 1;
                if (seg_first && i > 0) tc::mbar_wait(&bars->acc_empty, (seg - 1) & 1);
                tc::mbar_wait(&bars->i8_full[s], (i >> 1) & 1);
                tc::fence_after();
                const uint32_t a0 = tc::smem_u32(i8s + s * kI8Stage);
                const uint32_t b0 = a0 + tc::kDigits * kAPlane;
                // A plane b (high digit first, so the first MMA of a segment
                // initialises every diagonal) x B planes 5 - b .. 5 -> diagonals 5 .. 5 + b
#pragma unroll
                for (int b = tc::kDigits - 1; b >= 0; b--) {
                    const int ntot = (b + 1) * kWgN;
                    const int n1 = ntot <= 256 ? ntot : ((ntot / 2 + kWgN - 1) / kWgN) * kWgN;
                    const uint64_t ad = tc::smem_desc(a0 + b * kAPlane, kALbo, kGrpStride);
                    const uint32_t bs = b0 + (tc::kDigits - 1 - b) * kBPlane;
                    const uint32_t acc = (seg_first && b == tc::kDigits - 1) ? 0u : 1u;
                    tc::mma_i8(tmem, ad, tc::smem_desc(bs, kBLbo, kGrpStride), tc::idesc_i8_mn(kWgM, n1), acc);
                    if (n1 < ntot)
                        tc::mma_i8(tmem + n1, ad, tc::smem_desc(bs + (n1 / 16) * kGrpStride, kBLbo, kGrpStride),
                                   tc::idesc_i8_mn(kWgM, ntot - n1), acc);
                }
                tc::mma_commit(&bars->i8_empty[s]);
                if (seg_last) {
                    tc::mma_commit(&bars->acc_full);
                    seg++;
                }
            }
        }
    } else {
        // ---------------- converters + epilogue
        const int c = tid - 64, wi = c >> 5;
        const int q = warp & 3, colq = (warp - 2) >> 2;  // TMEM lane quarter, column quarter of the epilogue
        const int m = q * 32 + lane;                      // epilogue row (gate column within the half)
        const double sb = s_sb;
        // A: lane = 4 columns (conflict-free plane stores), rows wi + 16j
        const int m0 = lane * 4;
        const double sa0 = s_sa[m0], sa1 = s_sa[m0 + 1], sa2 = s_sa[m0 + 2], sa3 = s_sa[m0 + 3];
        // B (h part): row pairs (kb, kb + 4) per warp-iteration: lanes 0-15 /
        // 16-31, lane = 4 h columns (conflict-free with the 144 B group stride)
        const int hn0 = (lane & 15) * 4;
        const int hk = (wi & 3) + 8 * (wi >> 2) + 4 * (lane >> 4);
        RowPos hpos;
        hpos.init(step0 * kWgK + hk, T);
        // B (one-hot part): threads c < 128: row c / 4, 4-column group c % 4
        const int ok_ = c >> 2, og = c & 3;
        RowPos opos;
        opos.init(step0 * kWgK + ok_, T);
        int seg = 0;
        for (int i = 0; i < nsteps; i++) {
            const int s = i & 1;
            const int rb = (step0 + i) * kWgK;
            // per-row advantages / previous choices (global, L1): issued before the waits
            const double hw = rb + hk < rows ? (adv ? adv[hpos.q] : 1.0) : 0.0;
            double ow = 0.0;
            int prev = -1;
            if (c < 4 * kWgK) {
                const int row = rb + ok_;
                if (row < rows) {
                    ow = adv ? adv[opos.q] : 1.0;
                    prev = opos.r == 0 ? D : (int)choice[row - 1];
                }
            }
            const int hs0 = 2 * i, sl0 = hs0 % kSlots, sl1 = (hs0 + 1) % kSlots;
            tc::mbar_wait(&bars->f64_full[sl0], (hs0 / kSlots) & 1);
            tc::mbar_wait(&bars->f64_full[sl1], ((hs0 + 1) / kSlots) & 1);
            if (i >= 2) tc::mbar_wait(&bars->i8_empty[s], ((i - 2) >> 1) & 1);
            const uint8_t *slot0 = f64s + sl0 * kF64Slot, *slot1 = f64s + sl1 * kF64Slot;
            uint8_t *pa = i8s + s * kI8Stage;
            uint8_t *pb = pa + tc::kDigits * kAPlane;
            if (!(dbg & 1)) {
#pragma unroll
            for (int j = 0; j < 2; j++) {
                const int k = wi + 16 * j;
                const double *tda = reinterpret_cast<const double *>(j == 0 ? slot0 : slot1) + wi * kWgM + m0;
                const double2 x01 = *reinterpret_cast<const double2 *>(tda);
                const double2 x23 = *reinterpret_cast<const double2 *>(tda + 2);
                unsigned long long u[4];
                u[0] = tc::digits6(x01.x, sa0);
                u[1] = tc::digits6(x01.y, sa1);
                u[2] = tc::digits6(x23.x, sa2);
                u[3] = tc::digits6(x23.y, sa3);
                store_digits4(pa, kAPlane, plane_off(k, m0, kALbo), u);
            }
            {
                const int k = hk;
                const double *src = hpos.r == 0
                                        ? s_enc + hn0
                                        : reinterpret_cast<const double *>((k < kSlotRows ? slot0 : slot1) + kDaSlot) + (k & 15) * kH + hn0;
                const double2 x01 = *reinterpret_cast<const double2 *>(src);
                const double2 x23 = *reinterpret_cast<const double2 *>(src + 2);
                const double w = hw;
                unsigned long long u[4];
                u[0] = tc::digits6(x01.x * w, sb);
                u[1] = tc::digits6(x01.y * w, sb);
                u[2] = tc::digits6(x23.x * w, sb);
                u[3] = tc::digits6(x23.y * w, sb);
                store_digits4(pb, kBPlane, plane_off(k, hn0, kBLbo), u);
            }
            if (c < 4 * kWgK) {
                // one nonzero per row: adv at column 64 + prev (columns > 64 + D stay 0)
                const unsigned long long d = tc::digits6(ow, sb);
                const int sh = prev - 4 * og;
                const bool hit = sh >= 0 && sh < 4;
                const int off = plane_off(ok_, kH + 4 * og, kBLbo);
#pragma unroll
                for (int p = 0; p < 6; p++)
                    *reinterpret_cast<uint32_t *>(pb + p * kBPlane + off) =
                        hit ? (uint32_t)((d >> (8 * p)) & 0xFF) << (8 * sh) : 0u;
            }
            }
            tc::fence_async_smem();
            __syncwarp();
            if (lane == 0) {
                tc::mbar_arrive(&bars->f64_empty[sl0]);
                tc::mbar_arrive(&bars->f64_empty[sl1]);
                tc::mbar_arrive(&bars->i8_full[s]);
            }
            hpos.advance(T);
            opos.advance(T);
            const bool seg_last = i % seg_steps == seg_steps - 1 || i == nsteps - 1;
            if (seg_last) {
                // drain the 6 diagonal accumulators of this warp's lanes / columns
                tc::mbar_wait(&bars->acc_full, seg & 1);
                tc::fence_after();
                const uint32_t base = tmem + ((uint32_t)(q * 32) << 16) + colq * kEpCols;
                double acc[kEpCols];
#pragma unroll
                for (int j = 0; j < kEpCols; j++) acc[j] = 0.0;
#pragma unroll
                for (int e = tc::kDiags - 1; e >= 0; e--) {
                    const double wgt = tc::pow2(8 * (e + tc::kMinDiag));
                    uint32_t v[kEpCols];
                    tc::tmem_ld8(base + e * kWgN, *reinterpret_cast<uint32_t(*)[8]>(v));
                    tc::tmem_ld8(base + e * kWgN + 8, *reinterpret_cast<uint32_t(*)[8]>(v + 8));
                    tc::tmem_ld4(base + e * kWgN + 16, *reinterpret_cast<uint32_t(*)[4]>(v + 16));
                    tc::tmem_ld_wait();
#pragma unroll
                    for (int j = 0; j < kEpCols; j++) acc[j] = fma((double)(int)v[j], wgt, acc[j]);
                }
                // C[m][n] = acc * 2^-s_m * 2^-s_b -> partial[n][half * 128 + m] (first
                // segment stores, later ones add: one owner per element)
                const double inv = (1.0 / s_sa[m]);
                double *dst = partial + (size_t)chunk * part_stride + half * kWgM + m;
#pragma unroll
                for (int j = 0; j < kEpCols; j++) {
                    const int n = colq * kEpCols + j;
                    if (n < kH + D + 1) {
                        const double v = (acc[j] * inv) / sb;
                        dst[(size_t)n * kG] = seg ? dst[(size_t)n * kG] + v : v;
                    }
                }
                tc::fence_before();
                __syncwarp();
                if (lane == 0) tc::mbar_arrive(&bars->acc_empty);
                seg++;
            }
        }
    }
    tc::fence_before();
    __syncthreads();
    if (warp == 0) {
        tc::fence_after();
        tc::tmem_dealloc(tmem, kTmemCols);
    }
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

// row-major fp64 matrix [rows][cols] as a 2-D tensor map with box [box_rows][box_cols]
bool make_map(CUtensorMap *m, const double *base, int cols, int rows, int box_cols, int box_rows) {
    auto fn = encode_fn();
    if (!fn) return false;
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)cols * sizeof(double)};
    cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
    cuuint32_t es[2] = {1, 1};
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double *>(base), dims, strides, box, es,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

bool dec_wgrad_tc_ok(const PolicyDims &dm) { return dm.D + 1 + kH <= kWgN && encode_fn() != nullptr; }

int dec_wgrad_tc_chunks(int rows) {
    const int steps = (rows + kWgK - 1) / kWgK;
    const int n = steps < kNumSMs / 2 ? steps : kNumSMs / 2;
    return (steps + ceil_div(steps, n) - 1) / ceil_div(steps, n);
}

// partial[chunk][(64 + D + 1) x 256] like dec_wgrad_kernel; returns the chunk count via *n_chunks
int launch_dec_wgrad_tc(const PolicyDims &dm, int rows, const double *act_h, const double *enc_h,
                        const uint8_t *choice, const double *da, const int *colexp, const double *adv, int K,
                        double *partial, int *n_chunks, cudaStream_t st) {
    const int steps = (rows + kWgK - 1) / kWgK;
    const int n = steps < kNumSMs / 2 ? steps : kNumSMs / 2;
    const int per = ceil_div(steps, n);
    const int chunks = ceil_div(steps, per);
    CUtensorMap mda, mh;
    if (!make_map(&mda, da, kG, rows, kWgM, kSlotRows) || !make_map(&mh, act_h, kH, rows, kH, kSlotRows)) {
        set_error("cuTensorMapEncodeTiled failed");
        return DP_ECUDA;
    }
    DP_CUDA_TRY(cudaFuncSetAttribute(dec_wgrad_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kWgSmem));
    dec_wgrad_tc_kernel<<<2 * chunks, kWgThreads, kWgSmem, st>>>(
        mda, mh, dm.T, dm.D, rows, per, enc_h + (size_t)(dm.T - 1) * kH, choice, adv, K, colexp, partial,
        (size_t)(kH + dm.D + 1) * kG, dp_tensor_core_mode() == 2 ? 3 : kWgSeg,
        dp_tensor_core_mode() >= 3 ? dp_tensor_core_mode() - 2 : 0);
    DP_LAUNCH_CHECK();
    *n_chunks = chunks;
    return DP_OK;
}

}  // namespace dp
