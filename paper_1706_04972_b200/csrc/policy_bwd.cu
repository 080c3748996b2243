// Policy-gradient backward on sm_100a: grad = sum_k adv[k] * d log p_k / d theta.
//
// Reference: grad_log_prob (/root/reference/pkg/src/devplace/policy.py:351-409,
// _lstm_backward 236-253) called per sample by reinforce_update
// (pkg/trainer.py:138-154), which forms sum_k (r_k - b) * g_k.
//
// Restructuring — every step is linear in the per-sample
// advantage, so adv[k] scales dz at the top and all cross-sample sums happen
// inside the kernels:
//   B0 row_prep    (row tiles, fp64 micro-GEMMs): dz, du, dhc -> dh_out, dctx;
//                  q = W_att^T h; w = ctx.dctx (== alpha.dalpha); grads of
//                  b_out, dev_table[:D] (dz x u), w_out (hc x du)
//   B1 att_bwd     (row tiles x T-chunks): recompute s, alpha (forward softmax
//                  stats), dalpha = enc.dctx, ds = alpha*(dalpha - w);
//                  dq += ds@enc; d_enc += alpha^T dctx + ds^T q  (== d_enc +
//                  d_proj@W_att of the reference, proj@h restated as enc@(W_att^T h))
//   B1f row_fin    (row tiles): dh_ext = dh_out + dq@W_att^T; w_att grad += h^T dq
//   B2 lstm_bwd    (sequential over t, parallel over samples): LSTM backward,
//                  dh_prev = W_dec[dd:] da; da stored per row (in place)
//   B3 dec_wgrad   (row tiles, split-K): w_dec[dd:] += h_prev^T da; per input
//                  row sums of da give b_dec, w_dec[:dd] and dev_table row grads
//   B4 lstm_bwd    (sequential, ONE sequence): the encoder is shared by all
//                  samples, so its backward runs once on the summed inputs
//                  (the reference runs it per sample)
//   B5 enc_wgrad   w_enc, b_enc, type_table (np.add.at order)
// Deterministic: fixed partitions + ordered reductions.  The only float atomics
// (att_bwd's RED adds into per-sample partials) have a single writer per
// address per launch, so their result does not depend on scheduling.
// Measured B200 latencies that shaped the code (scripts/lat_probe.cu): DFMA
// ~8 cycles, LDS ~47, shfl ~27, exp ~160, tanh ~290: inner products use
// register micro-tiles (many independent FMAs per shared-memory load).

#include <math.h>

#include "fastmath.cuh"
#include "cpasync.cuh"
#include "policy.cuh"

namespace dp {

#define DP_TRY(x)                       \
    do {                                \
        const int rc_ = (x);            \
        if (rc_ != DP_OK) return rc_;   \
    } while (0)

static int g_tc_mode = 0;  // dp_debug_tensor_core
int dp_tensor_core_mode() { return g_tc_mode; }

namespace {

constexpr int kTile = 32;   // rows per tile (B0, B1, B3)
// Backward phases: kFused = one pass with the advantages; kRowsOnly = the
// advantage-independent per-row half (runs concurrently with the simulator);
// kGradsOnly = the advantage-weighted cross-row sums.
constexpr int kFused = 0, kRowsOnly = 1, kGradsOnly = 2;
constexpr int kFusedGrads = 3;  // B1f in the fused pass: grads only, rows already scaled (att_bwd did dh_ext)
constexpr int kFinTile = 64;
constexpr int kChunk = 64;  // B1: enc rows per chunk
constexpr int kPad = 65;

__device__ int g_att_dbg = 0;             // debug-only phase clocks of att_bwd (block 0, thread 0)
__device__ long long g_att_clk[8];

// ------------------------------------------------------------------ fp64 tensor core
// mma.sync m8n8k4 f64 (DMMA): D[8x8] += A[8x4] B[4x8], one warp.  Fragments
// (lane = 4 g + t): a = A[g][t], b = B[t][g], c/d = {C[g][2t], C[g][2t+1]}.
__device__ __forceinline__ void dmma884(double (&d)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d[0]), "+d"(d[1])
                 : "d"(a), "d"(b));
}

// ------------------------------------------------------------------ B0
// partial per CTA: [b_out (D) | dev_table[:D] (D*dd) | w_out (128*dd)]
// Operand tiles of the DMMA products use row strides == 8 (mod 32) words
// (68 / 132 / 36 doubles): the 4 k-rows x 8 lanes of a fragment load hit each
// bank pair at most twice (2 wavefronts for 256 bytes, the minimum).
constexpr int kPadH = 68, kWoLd = 2 * kH + 4, kDuLd = kMaxDD + 4;
struct PrepSmem {
    double watt[kH * kPadH];        // W_att[l][j]
    double woutT[kMaxDD * kWoLd];   // W_out^T [o][i]  (rows o >= dd zero)
    double devt[kMaxD * kMaxDD];    // dev_table[:D] [d][o]
    // cp.async double buffer of the tile's row operands (raw copies)
    double h[2][kTile * kPadH];     // [r][l]
    double uc[2][kTile * kMaxDD];   // ctx @ W_out[64:], rows of dd
    double u[2][kTile * kMaxDD];    // rows of dd
    double p[2][kTile * kMaxD];     // rows of D
    double w[2][kTile];             // per-row advantage (grads modes)
    uint8_t ch[2][kTile];
    double du[kTile * kDuLd];       // (cols >= dd zero)
    double dz[kTile * (kMaxD + 1)];
};

__global__ void __launch_bounds__(kThreads) row_prep_kernel(
    PolicyDims dm, const double *__restrict__ P, int rows, int tiles_per_cta, const double *__restrict__ adv,
    const double *__restrict__ act_p, const uint8_t *__restrict__ choice, const double *__restrict__ act_u,
    const double *__restrict__ act_h, const double *__restrict__ act_uc, double *__restrict__ row_q,
    double *__restrict__ row_w, double *__restrict__ row_dhx,
    double *__restrict__ row_du, double *__restrict__ partial,
    int mode /* kFused | kRowsOnly (adv := 1) | kGradsOnly */, int want_q /* 0: the attention backward runs in GM */) {
    extern __shared__ __align__(16) double smraw[];
    PrepSmem &S = *reinterpret_cast<PrepSmem *>(smraw);
    const bool rows_out = mode != kGradsOnly, grads_out = mode != kRowsOnly;
    const int tid = threadIdx.x;
    const int D = dm.D, dd = dm.dd, T = dm.T;
    const int Dp = D + 1;
    const int dd4 = (dd + 3) & ~3;  // DMMA k extent of the du @ W_out^T product
    const int n_tiles = (rows + kTile - 1) / kTile;
    const int t0 = blockIdx.x * tiles_per_cta, t1 = min(n_tiles, t0 + tiles_per_cta);
    // tile tl's rows -> buffer b, all asynchronous (zero-filled past the end)
    auto stage = [&](int tl, int b) {
        const int rb = tl * kTile;
        for (int x = tid * 2; x < kTile * kH; x += kThreads * 2) {
            const int r = x >> 6, j = x & 63;
            const bool ok = rb + r < rows;
            cp_async16(&S.h[b][r * kPadH + j], act_h + (ok ? (size_t)rb * kH + x : 0), ok);
        }
        for (int x = tid; x < kTile * dd; x += kThreads) {
            const bool ok = rb + x / dd < rows;
            cp_async8(&S.u[b][x], act_u + (ok ? (size_t)rb * dd + x : 0), ok);
            cp_async8(&S.uc[b][x], act_uc + (ok ? (size_t)rb * dd + x : 0), ok);
        }
        for (int x = tid; x < kTile * D; x += kThreads) {
            const bool ok = rb + x / D < rows;
            cp_async8(&S.p[b][x], act_p + (ok ? (size_t)rb * D + x : 0), ok);
        }
        if (tid < kTile) {
            const int row = rb + tid;
            const bool ok = row < rows;
            if (grads_out) cp_async8(&S.w[b][tid], adv + (ok ? row / T : 0), ok);
        } else if (tid < kTile + kTile / 8) {
            const int q = tid - kTile, row = rb + 8 * q;
            if (row + 8 <= rows) {
                cp_async8(&S.ch[b][8 * q], choice + row, true);
            } else {
                for (int e = 0; e < 8; e++) S.ch[b][8 * q + e] = row + e < rows ? choice[row + e] : 0;
            }
        }
        cp_async_commit();
    };
    if (t0 < t1) stage(t0, 0);
    for (int x = tid; x < kH * kH; x += kThreads) S.watt[(x >> 6) * kPadH + (x & 63)] = P[dm.off.w_att + x];
    for (int x = tid; x < 2 * kH * dd4; x += kThreads) {
        const int i = x / dd4, o = x % dd4;
        S.woutT[o * kWoLd + i] = o < dd ? P[dm.off.w_out + (size_t)i * dd + o] : 0.0;
    }
    for (int x = tid; x < D * dd; x += kThreads) S.devt[x] = P[dm.off.dev_table + x];
    // owned grad accumulators
    const int gi = tid >> 2, go = tid & 3;  // w_out grad (h rows): row i = gi, cols o = go + 4x
    double gw[kMaxDD / 4];
#pragma unroll
    for (int x = 0; x < kMaxDD / 4; x++) gw[x] = 0.0;
    double gdev[4] = {0.0, 0.0, 0.0, 0.0};  // dev grad: e = tid + 256*y < D*dd
    double gb = 0.0;                         // b_out: tid < D
    for (int tl = t0; tl < t1; tl++) {
        const int rb = tl * kTile, b = (tl - t0) & 1;
        if (tl + 1 < t1) {
            stage(tl + 1, b ^ 1);  // the next tile lands while this one is processed
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncthreads();
        const double *Sh = S.h[b], *Su = S.u[b], *Suc = S.uc[b];
        for (int x = tid; x < kTile * D; x += kThreads) {
            const int r = x / D, d = x - r * D;
            double dz = 0.0;
            if (rb + r < rows) {
                dz = -S.p[b][x];
                if (d == S.ch[b][r]) dz += 1.0;
                if (grads_out) dz = S.w[b][r] * dz;
            }
            S.dz[r * Dp + d] = dz;
        }
        __syncthreads();
        // du = dev_table[:D]^T dz (columns dd..dd4 zero for the DMMA k padding)
        for (int x = tid; x < kTile * dd4; x += kThreads) {
            const int r = x / dd4, o = x % dd4;
            double v = 0.0;
            if (o < dd) {
                for (int d = 0; d < D; d++) v = fma(S.devt[d * dd + o], S.dz[r * Dp + d], v);
                if (rows_out && rb + r < rows) row_du[(size_t)(rb + r) * dd + o] = v;
            }
            S.du[r * kDuLd + o] = v;
        }
        if (rows_out && want_q) {
            // q = h W_att (== W_att^T h per row) on the fp64 tensor cores:
            // warp w: rows 8 (w >> 1) .., columns 32 (w & 1) .. (4 n-tiles)
            const int lane = tid & 31, w = tid >> 5, g = lane >> 2, t = lane & 3;
            const int mt = w >> 1, nb = (w & 1) * 4;
            double acc[4][2];
#pragma unroll
            for (int n = 0; n < 4; n++) acc[n][0] = acc[n][1] = 0.0;
#pragma unroll 4
            for (int ks = 0; ks < kH / 4; ks++) {
                const double a = Sh[(mt * 8 + g) * kPadH + ks * 4 + t];
#pragma unroll
                for (int n = 0; n < 4; n++) dmma884(acc[n], a, S.watt[(ks * 4 + t) * kPadH + (nb + n) * 8 + g]);
            }
            const int row = rb + mt * 8 + g;
            if (row < rows)
#pragma unroll
                for (int n = 0; n < 4; n++)
                    *reinterpret_cast<double2 *>(row_q + (size_t)row * kH + (nb + n) * 8 + 2 * t) =
                        make_double2(acc[n][0], acc[n][1]);
        }
        __syncthreads();
        // dh_out = W_out[:64] du (DMMA, k = dd4).  The context half W_out[64:] du
        // is never formed: att_bwd contracts du with encW = enc W_out[64:].
        if (rows_out) {
            const int lane = tid & 31, w = tid >> 5, g = lane >> 2, t = lane & 3;
            const int mt = w >> 1, nb = (w & 1) * 4;
            double acc[4][2];
#pragma unroll
            for (int n = 0; n < 4; n++) acc[n][0] = acc[n][1] = 0.0;
            for (int ks = 0; ks < dd4 / 4; ks++) {
                const double a = S.du[(mt * 8 + g) * kDuLd + ks * 4 + t];
#pragma unroll
                for (int n = 0; n < 4; n++) dmma884(acc[n], a, S.woutT[(ks * 4 + t) * kWoLd + (nb + n) * 8 + g]);
            }
            const int row = rb + mt * 8 + g;
            if (row < rows)
#pragma unroll
                for (int n = 0; n < 4; n++)
                    *reinterpret_cast<double2 *>(row_dhx + (size_t)row * kH + (nb + n) * 8 + 2 * t) =
                        make_double2(acc[n][0], acc[n][1]);
        }
        // w = ctx . dctx == (ctx W_out[64:]) . du = uc . du  (8 lanes per row)
        if (rows_out) {
            const int r = tid >> 3, jb = tid & 7;
            double s0 = 0.0, s1 = 0.0;
#pragma unroll
            for (int x = 0; x < kMaxDD / 8; x += 2) {
                const int o0 = jb + 8 * x, o1 = o0 + 8;
                if (o0 < dd) s0 = fma(Suc[r * dd + o0], S.du[r * kDuLd + o0], s0);
                if (o1 < dd) s1 = fma(Suc[r * dd + o1], S.du[r * kDuLd + o1], s1);
            }
            double s = s0 + s1;
            s += __shfl_xor_sync(0xffffffffu, s, 1);
            s += __shfl_xor_sync(0xffffffffu, s, 2);
            s += __shfl_xor_sync(0xffffffffu, s, 4);
            const int row = rb + r;
            if (rows_out && jb == 0 && row < rows) row_w[row] = s;
        }
        if (grads_out) {
            // grads over the tile's rows (w_out h-half; the ctx half is enc^T A, att_fin_kernel)
            for (int r = 0; r < kTile; r++) {
                const double hc = Sh[r * kPadH + gi];
#pragma unroll
                for (int x = 0; x < kMaxDD / 4; x++) {
                    const int o = go + 4 * x;
                    if (o < dd) gw[x] = fma(hc, S.du[r * kDuLd + o], gw[x]);
                }
            }
#pragma unroll
            for (int y = 0; y < 4; y++) {
                const int e = tid + kThreads * y;
                if (e < D * dd) {
                    const int d = e / dd, o = e % dd;
                    double v = gdev[y];
                    for (int r = 0; r < kTile; r++) v = fma(S.dz[r * Dp + d], Su[r * dd + o], v);
                    gdev[y] = v;
                }
            }
            if (tid < D)
                for (int r = 0; r < kTile; r++) gb += S.dz[r * Dp + tid];
        }
        __syncthreads();  // buffer b and du / dz are rewritten next iteration
    }
    if (!grads_out) return;
    const size_t na = (size_t)D + D * dd + 2 * kH * dd;
    double *out = partial + (size_t)blockIdx.x * na;
    if (tid < D) out[tid] = gb;
#pragma unroll
    for (int y = 0; y < 4; y++) {
        const int e = tid + kThreads * y;
        if (e < D * dd) out[D + e] = gdev[y];
    }
#pragma unroll
    for (int x = 0; x < kMaxDD / 4; x++) {
        const int o = go + 4 * x;
        if (o < dd) out[D + D * dd + gi * dd + o] = gw[x];
    }
}

// ------------------------------------------------------------------ B0g / B1fg
// Advantage-weighted halves of B0 and B1f in the split backward (dz0 =
// onehot(choice) - p, du0 = dev_table[:D]^T dz0 from the rows pass):
// one pass over the rows computes every advantage-weighted
// output-side gradient,
//   [w_att | w_out[:64]] += (adv o H)^T [DQ | DU]     (64 x (64 + dd), DMMA)
//   dev_table          += (adv o DZ)^T U            (D x dd, SIMT)
//   b_out              += sum_r adv_r dz[r]
// with dz = onehot(choice) - p.  32-row tiles of h and [dq | du] stream through
// a cp.async double buffer (row strides == 8 mod 32 words: conflict-free
// fragment loads); warp w owns m-tile w (h units 8w..8w+7) x all n-tiles.
// partial per CTA: [b_out D | dev_table D*dd | w_out[:64] 64*dd | w_att 64*64].
constexpr int kAgLdH = kH + 4, kAgLdB = kH + kMaxDD + 4, kAgNt = (kH + kMaxDD) / 8;
struct AdvGradSmem {
    double h[2][kTile][kAgLdH];
    double b[2][kTile][kAgLdB];      // [dq (64) | du (dd) | 0]
    double u[2][kTile][kMaxDD];
    double p[2][kTile][kMaxD];
    double w[2][kTile];
    uint8_t ch[2][kTile];
};
__host__ __device__ inline size_t adv_grads_partial(const PolicyDims &dm) {
    return (size_t)dm.D + dm.D * dm.dd + kH * dm.dd + kH * kH;
}
__global__ void __launch_bounds__(kThreads, 1) adv_grads_kernel(PolicyDims dm, int rows, int tiles_per_cta,
                                                                const double *__restrict__ adv,
                                                                const double *__restrict__ act_h,
                                                                const double *__restrict__ row_dq,
                                                                const double *__restrict__ row_du,
                                                                const double *__restrict__ act_u,
                                                                const double *__restrict__ act_p,
                                                                const uint8_t *__restrict__ choice,
                                                                double *__restrict__ partial,
                                                                int nq /* dq columns: 64, or 0 when the grads pass forms W_att from G */) {
    extern __shared__ __align__(16) double sm_raw[];
    AdvGradSmem &S = *reinterpret_cast<AdvGradSmem *>(sm_raw);
    const int tid = threadIdx.x, lane = tid & 31, wp = tid >> 5, g = lane >> 2, t = lane & 3;
    const int T = dm.T, D = dm.D, dd = dm.dd;
    const int nt_used = (nq + dd + 7) / 8;
    double acc[kAgNt][2];
#pragma unroll
    for (int n = 0; n < kAgNt; n++) acc[n][0] = acc[n][1] = 0.0;
    double gdev = 0.0, gb = 0.0;  // thread tid < D*dd: dev_table[d][o]; tid < D: b_out[d]
    const int dv_d = tid / (dd > 0 ? dd : 1), dv_o = tid - dv_d * dd;
    const int n_tiles = (rows + kTile - 1) / kTile;
    const int t0 = blockIdx.x * tiles_per_cta, t1 = min(n_tiles, t0 + tiles_per_cta);
    // zero the padding columns of both B buffers once (never written by the copies)
    const int npad = kAgLdB - nq - dd;
    for (int x = tid; x < 2 * kTile * npad; x += kThreads) {
        const int bb = x / (kTile * npad), rem = x - bb * kTile * npad;
        const int r = rem / npad, c = rem - r * npad;
        S.b[bb][r][nq + dd + c] = 0.0;
    }
    auto stage = [&](int tl, int bf) {
        const int rb = tl * kTile;
        for (int x = tid * 2; x < kTile * kH; x += kThreads * 2) {
            const int r = x >> 6, c = x & 63;
            const bool ok = rb + r < rows;
            cp_async16(&S.h[bf][r][c], act_h + (ok ? (size_t)rb * kH + x : 0), ok);
            if (nq) cp_async16(&S.b[bf][r][c], row_dq + (ok ? (size_t)rb * kH + x : 0), ok);
        }
        // the small per-row operands also go asynchronously (8-byte copies; a
        // plain load would stall this thread before the current tile's math)
        for (int x = tid; x < kTile * dd; x += kThreads) {
            const int r = x / dd, c = x - r * dd;
            const bool ok = rb + r < rows;
            cp_async8(&S.b[bf][r][nq + c], row_du + (ok ? (size_t)rb * dd + x : 0), ok);
            cp_async8(&S.u[bf][r][c], act_u + (ok ? (size_t)rb * dd + x : 0), ok);
        }
        for (int x = tid; x < kTile * D; x += kThreads) {
            const int r = x / D;
            const bool ok = rb + r < rows;
            cp_async8(&S.p[bf][r][x - r * D], act_p + (ok ? (size_t)rb * D + x : 0), ok);
        }
        if (tid < kTile) {
            const int row = rb + tid;
            const bool ok = row < rows;
            cp_async8(&S.w[bf][tid], adv + (ok ? row / T : 0), ok);
        } else if (tid < kTile + kTile / 8) {
            // choices: 8-byte words of the tile's 32 bytes (rows are 32-aligned)
            const int q = tid - kTile, row = rb + 8 * q;
            if (row + 8 <= rows) {
                cp_async8(&S.ch[bf][8 * q], choice + row, true);
            } else {
                for (int e = 0; e < 8; e++) S.ch[bf][8 * q + e] = row + e < rows ? choice[row + e] : 0;
            }
        }
        cp_async_commit();
    };
    if (t0 < t1) stage(t0, 0);
    for (int tl = t0; tl < t1; tl++) {
        const int bf = (tl - t0) & 1;
        if (tl + 1 < t1) {
            stage(tl + 1, bf ^ 1);
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncthreads();
#pragma unroll 2
        for (int ks = 0; ks < kTile / 4; ks++) {
            const int r = ks * 4 + t;
            const double a = S.h[bf][r][wp * 8 + g] * S.w[bf][r];
#pragma unroll
            for (int n = 0; n < kAgNt; n++)
                if (n < nt_used) dmma884(acc[n], a, S.b[bf][r][n * 8 + g]);
        }
        if (tid < D * dd) {
            double v0 = 0.0, v1 = 0.0;
#pragma unroll 4
            for (int r = 0; r < kTile; r += 2) {
                const double z0 = (S.ch[bf][r] == dv_d ? 1.0 : 0.0) - S.p[bf][r][dv_d];
                const double z1 = (S.ch[bf][r + 1] == dv_d ? 1.0 : 0.0) - S.p[bf][r + 1][dv_d];
                v0 = fma(S.w[bf][r] * z0, S.u[bf][r][dv_o], v0);
                v1 = fma(S.w[bf][r + 1] * z1, S.u[bf][r + 1][dv_o], v1);
            }
            gdev += v0 + v1;
        }
        if (tid < D) {
            double v = 0.0;
            for (int r = 0; r < kTile; r++)
                v = fma(S.w[bf][r], (S.ch[bf][r] == tid ? 1.0 : 0.0) - S.p[bf][r][tid], v);
            gb += v;
        }
        __syncthreads();  // buffer bf is re-staged by the next iteration
    }
    double *out = partial + (size_t)blockIdx.x * adv_grads_partial(dm);
    if (tid < D) out[tid] = gb;
    if (tid < D * dd) out[D + tid] = gdev;
    double *o1 = out + D + D * dd, *oa = o1 + kH * dd;
    const int l = wp * 8 + g;
#pragma unroll
    for (int n = 0; n < kAgNt; n++)
#pragma unroll
        for (int e = 0; e < 2; e++) {
            const int c = n * 8 + 2 * t + e;
            if (c < nq) oa[l * kH + c] = acc[n][e];
            else if (c < nq + dd) o1[l * dd + (c - nq)] = acc[n][e];
        }
}

// ------------------------------------------------------------------ B1
constexpr int kAttTile = 64;  // rows per tile in att_bwd (2 rows per thread in the S/DA and dq passes)
// GM prep scratch: uc rows [64][dd] at S.al[0], p rows [64][D] at S.al[kPrepP];
// W_out[:64]^T [dd4][kPadH] at S.ds[0], dev_table [D][dd] at S.ds[kPrepDev]
constexpr int kPrepP = kAttTile * kMaxDD, kPrepDev = kMaxDD * 68;

struct AttSmem {
    double enc[2][kChunk * kPadH];  // cp.async double buffer over the T chunks
    double encw[2][kChunk * kDuLd]; // encW = enc W_out[64:] rows of the chunk (cols >= dd zero)
    double q[kAttTile * kPadH];
    double al[kAttTile * kPadH];
    double ds[kAttTile * kPadH];
    double du[kAttTile * kDuLd];
    double mx[kAttTile], sm[kAttTile], w[kAttTile];
};

// Tile-outer: a CTA owns whole 64-step tiles of one sample; per tile its
// q / dctx / du / stats are staged once, the 64-row chunks of enc_states
// stream through a cp.async double buffer, and dq accumulates in registers
// over the chunks (one store per tile).  Every contraction is a 64x64x64 (or
// 64 x dd x 64) product on the fp64 tensor cores (mma.sync m8n8k4 DMMA);
// warp w owns the 8-row m-tile w of each product:
//   DA    dalpha[r, i] = dctx[r] . enc_i = du[r] . encW_i   (dctx = W_out[64:] du, so a
//         k = dd product on encW = enc W_out[64:] from the forward; S = q . enc_i too,
//         unless STORED)
//         alpha (STORED: e_i * esc from the decoder; else exp(s - max) / sum),
//         ds = alpha (dalpha - w)
//   dq    += ds @ enc_chunk
//   dE    d_enc[i, j] = sum_r ds[r, i] q[r, j],  A[i, o] = sum_r alpha[r, i] du[r, o]
// dE / A go to the per-sample (or per-tile) partials of the split backward,
// or accumulate in the CTA's private partial (fused backward).
// GM (split backward with stored numerators): the launch passes proj for
// enc_h and act_h for row_q, so the same products give dh_ext = ds proj
// (instead of dq; dh_ext = dq W_att^T = ds enc W_att^T) and the per-sample
// G = ds^T H (instead of d_enc = ds^T q = G W_att); the grads pass forms
// d_enc = (sum adv G) W_att and dW_att = (sum adv G)^T enc once.  No dh_ext
// epilogue product, no row_dq.
template <bool STORED, bool GM = false>
__global__ void __launch_bounds__(kThreads, 1) att_bwd_kernel(
    PolicyDims dm, int rows, int tiles_per_cta, const double *__restrict__ enc_h,
    const double *__restrict__ act_stat, const double *__restrict__ row_q, const double *__restrict__ encW,
    const double *__restrict__ row_w, const double *__restrict__ row_du, double *__restrict__ row_dq,
    double *__restrict__ partial, double *__restrict__ partA,
    double *__restrict__ tile_partial /* [units][T][64] or NULL */,
    double *__restrict__ tile_partA /* [units][T][dd] */, const double *__restrict__ act_e,
    const double *__restrict__ act_esc, int do_denc, int per_sample /* partials per sample, not per tile */,
    const double *__restrict__ w_att, double *__restrict__ row_dhx /* dh_ext += dq W_att^T (B1f rows part) */,
    // GM with prep: the rows pass's per-row half of B0 formed here per tile (no row_prep
    // launch): dz = onehot(choice) - p, du = dev_table[:D]^T dz (-> row_du_out), w = uc . du,
    // and dh_out = W_out[:64] du as the initial value of the tile's dh_ext accumulator
    int prep = 0, const double *__restrict__ P = nullptr, const double *__restrict__ act_p = nullptr,
    const uint8_t *__restrict__ choice = nullptr, const double *__restrict__ act_uc = nullptr,
    double *__restrict__ row_du_out = nullptr) {
    extern __shared__ __align__(16) double smraw[];
    AttSmem &S = *reinterpret_cast<AttSmem *>(smraw);
    const int tid = threadIdx.x, lane = tid & 31, wp = tid >> 5, g = lane >> 2, t = lane & 3;
    const int T = dm.T, dd = dm.dd;
    const int dd8 = (dd + 7) & ~7;  // n extent of the A product (8-column tiles)
    const int n_chunks = (T + kChunk - 1) / kChunk;
    const int tps = (T + kAttTile - 1) / kAttTile;
    const int tile0 = blockIdx.x * tiles_per_cta;
    const int n_tiles_total = (rows / T) * tps;
    const int tile1 = min(n_tiles_total, tile0 + tiles_per_cta);
    const int mr = wp * 8 + g;  // this lane's row of the m-tile (r for DA / dq, i for dE / A)
    // enc chunk c -> buffer b (16-byte cp.async; rows past T zero-filled)
    auto stage_enc = [&](int c, int b) {
        const int i0 = c * kChunk;
        for (int x = tid; x < kChunk * (kH / 2); x += kThreads) {
            const int i = x >> 5, j2 = x & 31;
            const bool ok = i0 + i < T;
            cp_async16(&S.enc[b][i * kPadH + 2 * j2], enc_h + (size_t)(ok ? i0 + i : 0) * kH + 2 * j2, ok);
        }
        for (int x = tid; x < kChunk * dd; x += kThreads) {
            const int i = x / dd;
            const bool ok = i0 + i < T;
            cp_async8(&S.encw[b][i * kDuLd + (x - i * dd)], encW + (ok ? (size_t)i0 * dd + x : 0), ok);
        }
        cp_async_commit();
    };
    // the tile's q / du / softmax stats -> shared memory (cp.async; du columns
    // dd..dd8 stay zero from the prologue), and this lane's 16 dctx values of
    // its DA rows -> registers (the A fragments of the DA product)
    auto stage_tile = [&](int tl) {
        const int t0 = (tl % tps) * kAttTile;
        const int rb = (tl / tps) * T + t0;
        const int nrow = min(kAttTile, T - t0);
        for (int x = tid * 2; x < kAttTile * kH; x += kThreads * 2) {
            const int r = x >> 6, j = x & 63;
            const bool ok = r < nrow;
            cp_async16(&S.q[r * kPadH + j], row_q + (ok ? (size_t)(rb + r) * kH + j : 0), ok);
        }
        if (GM && prep) {
            // the tile's uc / p rows into scratch (S.al is free until the first chunk's ds)
            for (int x = tid; x < kAttTile * dd; x += kThreads) {
                const bool ok = x / dd < nrow;
                cp_async8(&S.al[x], act_uc + (ok ? (size_t)rb * dd + x : 0), ok);
            }
            for (int x = tid; x < kAttTile * dm.D; x += kThreads) {
                const bool ok = x / dm.D < nrow;
                cp_async8(&S.al[kPrepP + x], act_p + (ok ? (size_t)rb * dm.D + x : 0), ok);
            }
        } else {
            for (int x = tid; x < kAttTile * dd; x += kThreads) {
                const int r = x / dd;
                const bool ok = r < nrow;
                cp_async8(&S.du[r * kDuLd + (x - r * dd)], row_du + (ok ? (size_t)rb * dd + x : 0), ok);
            }
        }
        if (tid < kAttTile) {
            const bool ok = tid < nrow;
            const size_t row = ok ? (size_t)(rb + tid) : 0;
            cp_async8(&S.mx[tid], act_stat + row * 2, ok);
            cp_async8(&S.sm[tid], act_stat + row * 2 + 1, ok);
            if (!(GM && prep)) cp_async8(&S.w[tid], row_w + row, ok);
        }
        cp_async_commit();
    };
    // zero k-padding columns (dd .. kDuLd) of du and of both encW buffers once:
    // the copies never write them
    for (int x = tid; x < kAttTile * (kDuLd - dd); x += kThreads) {
        const int r = x / (kDuLd - dd), c = dd + (x - r * (kDuLd - dd));
        S.du[r * kDuLd + c] = 0.0;
        S.encw[0][r * kDuLd + c] = 0.0;
        S.encw[1][r * kDuLd + c] = 0.0;
    }
    const int dd4 = (dd + 3) & ~3;  // k extent of the DA product
    if (tile0 < tile1) {
        stage_tile(tile0);
        stage_enc(0, 0);
    }
    const bool aclk = g_att_dbg && blockIdx.x == 0 && tid == 0;
    long long ac_last = aclk ? clock64() : 0, ac[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#define DP_APHASE(i)                        \
    if (aclk) {                             \
        const long long now_ = clock64();   \
        ac[i] += now_ - ac_last;            \
        ac_last = now_;                     \
    }
    bool first_cta_tile = true;
    for (int tl = tile0; tl < tile1; tl++) {
        const int t0 = (tl % tps) * kAttTile;
        const int rb = (tl / tps) * T + t0;
        const int nrow = min(kAttTile, T - t0);
        double dq[8][2];  // dq[mr][n*8 + 2t + {0,1}], accumulated over the chunks
#pragma unroll
        for (int n = 0; n < 8; n++) dq[n][0] = dq[n][1] = 0.0;
        const bool rok = mr < nrow;
        for (int ch = 0; ch < n_chunks; ch++) {
            const int i0 = ch * kChunk, b = ch & 1;
            // this lane's stored numerators (issued before the wait: the loads
            // overlap the chunk's cp.async and the DA product)
            double ev[8][2], esc0 = 0.0, esc1 = 0.0;
            if (STORED) {
                const size_t row = (size_t)(rb + (rok ? mr : 0));
#pragma unroll
                for (int n = 0; n < 8; n++) {
                    const int ig = i0 + n * 8 + 2 * t;
                    if (rok && ig + 1 < T && ((row * T) & 1) == 0) {  // 16-byte aligned pair
                        const double2 e2 = __ldg(reinterpret_cast<const double2 *>(act_e + row * T + ig));
                        ev[n][0] = e2.x;
                        ev[n][1] = e2.y;
                    } else {
                        ev[n][0] = (rok && ig < T) ? __ldg(act_e + row * T + ig) : 0.0;
                        ev[n][1] = (rok && ig + 1 < T) ? __ldg(act_e + row * T + ig + 1) : 0.0;
                    }
                }
                esc0 = __ldg(act_esc + row * 8 + ((i0 & 255) >> 5));
                esc1 = __ldg(act_esc + row * 8 + (((i0 + 32) & 255) >> 5));
            }
            if (ch + 1 < n_chunks) {
                stage_enc(ch + 1, b ^ 1);
                cp_async_wait<1>();
            } else {
                cp_async_wait<0>();
            }
            __syncthreads();
            if (GM && prep && ch == 0) {
                // B0's per-row half for this tile (row_prep_kernel's rows-only outputs)
                const int D = dm.D;
                const int dd4p = (dd + 3) & ~3;
                double *wT = S.ds;               // W_out[:64]^T [o][j], o < dd4p (S.ds is free here)
                double *dvt = S.ds + kPrepDev;   // dev_table[:D] [d][o]
                for (int x = tid; x < dd4p * kH; x += kThreads) {
                    const int j = x / dd4p, o = x - j * dd4p;  // o fastest: coalesced W_out rows
                    wT[o * kPadH + j] = o < dd ? __ldg(P + dm.off.w_out + (size_t)j * dd + o) : 0.0;
                }
                for (int x = tid; x < D * dd; x += kThreads) dvt[x] = __ldg(P + dm.off.dev_table + x);
                const int rb0 = (tl / tps) * T + (tl % tps) * kAttTile;
                const int nrow0 = min(kAttTile, T - (tl % tps) * kAttTile);
                __syncthreads();
                // du = dev_table[:D]^T dz, dz = onehot(choice) - p (row_prep's order)
                for (int x = tid; x < kAttTile * dd4p; x += kThreads) {
                    const int r = x / dd4p, o = x - r * dd4p;
                    double v = 0.0;
                    if (o < dd && r < nrow0) {
                        const int chr = choice[rb0 + r];
                        for (int d = 0; d < D; d++) {
                            double dz = -S.al[kPrepP + r * D + d];
                            if (d == chr) dz += 1.0;
                            v = fma(dvt[d * dd + o], dz, v);
                        }
                        row_du_out[(size_t)(rb0 + r) * dd + o] = v;
                    }
                    S.du[r * kDuLd + o] = v;
                }
                __syncthreads();
                // w = uc . du (8 lanes per row, two passes of 32 rows)
                for (int pass = 0; pass < 2; pass++) {
                    const int r = pass * 32 + (tid >> 3), jb = tid & 7;
                    double s0 = 0.0, s1 = 0.0;
#pragma unroll
                    for (int x = 0; x < kMaxDD / 8; x += 2) {
                        const int o0 = jb + 8 * x, o1 = o0 + 8;
                        if (o0 < dd) s0 = fma(S.al[r * dd + o0], S.du[r * kDuLd + o0], s0);
                        if (o1 < dd) s1 = fma(S.al[r * dd + o1], S.du[r * kDuLd + o1], s1);
                    }
                    double sw = s0 + s1;
                    sw += __shfl_xor_sync(0xffffffffu, sw, 1);
                    sw += __shfl_xor_sync(0xffffffffu, sw, 2);
                    sw += __shfl_xor_sync(0xffffffffu, sw, 4);
                    if (jb == 0) S.w[r] = r < nrow0 ? sw : 0.0;
                }
                // dh_out = W_out[:64] du as the dh_ext accumulator's start (DMMA, k = dd4p)
                for (int ks = 0; ks < dd4p / 4; ks++) {
                    const double a = S.du[mr * kDuLd + ks * 4 + t];
#pragma unroll
                    for (int n = 0; n < 8; n++) dmma884(dq[n], a, wT[(ks * 4 + t) * kPadH + n * 8 + g]);
                }
                __syncthreads();  // S.w / S.du complete; the scratch in S.al / S.ds is free again
            }
            DP_APHASE(0);
            const double *enc = S.enc[b];
            // DA (and S) for rows mr, columns i = n*8 + 2t + {0,1}
            {
                double da[8][2], sv[8][2];
#pragma unroll
                for (int n = 0; n < 8; n++) da[n][0] = da[n][1] = sv[n][0] = sv[n][1] = 0.0;
                const double *ew = S.encw[b];
                for (int ks = 0; ks < dd4 / 4; ks++) {
                    const double a = S.du[mr * kDuLd + ks * 4 + t];
#pragma unroll
                    for (int n = 0; n < 8; n++) dmma884(da[n], a, ew[(n * 8 + g) * kDuLd + ks * 4 + t]);  // B[o][i] = encW[i][o]
                }
                if (!STORED)
#pragma unroll
                    for (int ks = 0; ks < kH / 4; ks++) {
                        const double aq = S.q[mr * kPadH + ks * 4 + t];
#pragma unroll
                        for (int n = 0; n < 8; n++) dmma884(sv[n], aq, enc[(n * 8 + g) * kPadH + ks * 4 + t]);
                    }
                const double m = S.mx[mr], l = S.sm[mr], wv = S.w[mr];
                // score recompute: alpha = exp(s - max) / sum as branch-free fastmath
                // exp times one reciprocal per row (libm exp and 16 divisions per lane
                // serialised the chunk; both within a few ulp, far inside 1e-9)
                const double rl = STORED ? 0.0 : fm_rcp(l);
#pragma unroll
                for (int n = 0; n < 8; n++)
#pragma unroll
                    for (int e = 0; e < 2; e++) {
                        const int i = n * 8 + 2 * t + e;
                        double al = 0.0, dsv = 0.0;
                        if (i0 + i < T && rok) {
                            al = STORED ? ev[n][e] * (n < 4 ? esc0 : esc1) : fm_exp(sv[n][e] - m) * rl;
                            dsv = al * (da[n][e] - wv);
                        }
                        S.al[mr * kPadH + i] = al;
                        S.ds[mr * kPadH + i] = dsv;
                    }
            }
            DP_APHASE(1);
            __syncthreads();
            DP_APHASE(2);
            // dq[mr, j] += sum_i ds[mr, i] enc[i, j]
#pragma unroll 2
            for (int ks = 0; ks < kChunk / 4; ks++) {
                const double a = S.ds[mr * kPadH + ks * 4 + t];
#pragma unroll
                for (int n = 0; n < 8; n++) dmma884(dq[n], a, enc[(ks * 4 + t) * kPadH + n * 8 + g]);
            }
            DP_APHASE(3);
            if (!do_denc) {
                __syncthreads();
                continue;
            }
            // dE[i = mr, j] = sum_r ds[r, i] q[r, j] ; A[i = mr, o] = sum_r al[r, i] du[r, o]
            double dE[8][2], dA[4][2];
#pragma unroll
            for (int n = 0; n < 8; n++) dE[n][0] = dE[n][1] = 0.0;
#pragma unroll
            for (int n = 0; n < 4; n++) dA[n][0] = dA[n][1] = 0.0;
#pragma unroll 2
            for (int ks = 0; ks < kAttTile / 4; ks++) {
                const int r = ks * 4 + t;
                const double a = S.ds[r * kPadH + mr];
                const double aa = S.al[r * kPadH + mr];
#pragma unroll
                for (int n = 0; n < 8; n++) dmma884(dE[n], a, S.q[r * kPadH + n * 8 + g]);
#pragma unroll
                for (int n = 0; n < 4; n++)
                    if (n * 8 < dd8) dmma884(dA[n], aa, S.du[r * kDuLd + n * 8 + g]);
            }
            DP_APHASE(4);
            // every shared operand of this chunk is consumed: the barrier comes
            // before the partial stores (registers only), and after a tile's
            // last chunk (GM) the next tile's operands go out now, so they land
            // while the stores drain
            __syncthreads();  // al / ds / q / du / this enc buffer are overwritten next
            if (GM && ch == n_chunks - 1 && tl + 1 < tile1) {
                stage_tile(tl + 1);
                stage_enc(0, 0);
            }
            DP_APHASE(6);
            const int i = i0 + mr;
            if (i < T) {
                const size_t unit = per_sample ? (size_t)(tl / tps) : (size_t)tl;
                const bool first = tile_partial ? (!per_sample || tl % tps == 0) : first_cta_tile;
                double *pe = tile_partial ? tile_partial + (unit * T + i) * kH
                                          : partial + ((size_t)blockIdx.x * T + i) * kH;
                double *pa = tile_partial ? tile_partA + (unit * T + i) * dd : partA + ((size_t)blockIdx.x * T + i) * dd;
                // first contribution stores; later ones add with fire-and-forget
                // reductions (RED).  One thread owns each element and its
                // operations on one address stay in program order: deterministic.
#pragma unroll
                for (int n = 0; n < 8; n++)
#pragma unroll
                    for (int e = 0; e < 2; e++) {
                        double *d = pe + n * 8 + 2 * t + e;
                        if (first) *d = dE[n][e];
                        else atomicAdd(d, dE[n][e]);
                    }
#pragma unroll
                for (int n = 0; n < 4; n++)
#pragma unroll
                    for (int e = 0; e < 2; e++) {
                        const int o = n * 8 + 2 * t + e;
                        if (o < dd) {
                            if (first) pa[o] = dA[n][e];
                            else atomicAdd(pa + o, dA[n][e]);
                        }
                    }
            }
            DP_APHASE(5);
        }
        if (GM) {
            // dq holds ds proj = this tile's dh_ext contribution
            if (rok)
#pragma unroll
                for (int n = 0; n < 8; n++) {
                    double2 *dst = reinterpret_cast<double2 *>(row_dhx + (size_t)(rb + mr) * kH + n * 8 + 2 * t);
                    if (prep) {
                        *dst = make_double2(dq[n][0], dq[n][1]);  // dh_out + ds proj, formed here
                    } else {
                        const double2 v = *dst;
                        *dst = make_double2(v.x + dq[n][0], v.y + dq[n][1]);
                    }
                }
            first_cta_tile = false;
            DP_APHASE(7);
            continue;
        }
        if (rok)
#pragma unroll
            for (int n = 0; n < 8; n++)
                *reinterpret_cast<double2 *>(row_dq + (size_t)(rb + mr) * kH + n * 8 + 2 * t) =
                    make_double2(dq[n][0], dq[n][1]);
        // B1f rows part fused here: dh_ext[r, l] += sum_j dq[r, j] W_att[l, j]
        // (dq -> S.ds and W_att -> S.al, both free after the last chunk).  The
        // next tile's q / du / stats / first enc chunk are issued first, so they
        // land while this product runs.
#pragma unroll
        for (int n = 0; n < 8; n++) {
            S.ds[mr * kPadH + n * 8 + 2 * t] = dq[n][0];
            S.ds[mr * kPadH + n * 8 + 2 * t + 1] = dq[n][1];
        }
        if (tl + 1 < tile1) {
            stage_tile(tl + 1);
            stage_enc(0, 0);
        }
        for (int x = tid; x < kH * kH; x += kThreads) S.al[(x >> 6) * kPadH + (x & 63)] = __ldg(w_att + x);
        __syncthreads();
        {
            double o[8][2];
#pragma unroll
            for (int n = 0; n < 8; n++) o[n][0] = o[n][1] = 0.0;
#pragma unroll 2
            for (int ks = 0; ks < kH / 4; ks++) {
                const double a = S.ds[mr * kPadH + ks * 4 + t];
#pragma unroll
                for (int n = 0; n < 8; n++) dmma884(o[n], a, S.al[(n * 8 + g) * kPadH + ks * 4 + t]);
            }
            if (rok)
#pragma unroll
                for (int n = 0; n < 8; n++) {
                    double2 *dst = reinterpret_cast<double2 *>(row_dhx + (size_t)(rb + mr) * kH + n * 8 + 2 * t);
                    const double2 v = *dst;
                    *dst = make_double2(v.x + o[n][0], v.y + o[n][1]);
                }
        }
        __syncthreads();  // S.ds / S.al are rewritten by the next tile's first chunk
        first_cta_tile = false;
        DP_APHASE(7);
    }
#undef DP_APHASE
    if (aclk)
        for (int k = 0; k < 8; k++) g_att_clk[k] += ac[k];
}

// ------------------------------------------------------------------ B1g (GM)
// From G = sum_k adv_k ds_k^T H_k [T][64]:
//   blocks b < nb:  d_enc[i] = G[i] W_att for rows i = 4b .. 4b+3 (W_att and the
//                   rows staged in shared memory; att_fin adds the context part)
//   blocks nb + l:  grad W_att[l][:] = sum_i G[i][l] enc[i][:]  (4 row slices per
//                   column, fixed-order combine)
// plus the context part of B1a (att_fin_kernel, fused here): d_enc[i] +=
// A[i] W_out[64:]^T, and blocks nb + 64 + x: grad W_out[64:] = enc^T A.
constexpr int kGfRows = 4;
__global__ void __launch_bounds__(256) gsum_fin_kernel(PolicyDims dm, const double *__restrict__ P, int nb,
                                                       const double *__restrict__ G, const double *__restrict__ A,
                                                       const double *__restrict__ enc_h, double *__restrict__ d_enc,
                                                       double *__restrict__ grad) {
    const int T = dm.T, dd = dm.dd;
    const double *w_att = P + dm.off.w_att, *w2 = P + dm.off.w_out + (size_t)kH * dd;
    double *g_watt = grad + dm.off.w_att;
    __shared__ double wa[kH * kH];
    __shared__ double gr[kGfRows][kH];
    __shared__ double part[4][kH];
    const int tid = threadIdx.x, j = tid & 63, q = tid >> 6;
    if ((int)blockIdx.x < nb) {
        const int i0 = blockIdx.x * kGfRows;
        for (int x = tid; x < kH * kH; x += 256) wa[x] = w_att[x];
        const int i = i0 + q;
        gr[q][j] = i < T ? G[(size_t)i * kH + j] : 0.0;
        __syncthreads();
        double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
#pragma unroll
        for (int l = 0; l < kH; l += 4) {
            a0 = fma(gr[q][l], wa[l * kH + j], a0);
            a1 = fma(gr[q][l + 1], wa[(l + 1) * kH + j], a1);
            a2 = fma(gr[q][l + 2], wa[(l + 2) * kH + j], a2);
            a3 = fma(gr[q][l + 3], wa[(l + 3) * kH + j], a3);
        }
        double c0 = 0.0;
        if (i < T)
            for (int o = 0; o < dd; o++) c0 = fma(A[(size_t)i * dd + o], w2[(size_t)j * dd + o], c0);
        if (i < T) d_enc[(size_t)i * kH + j] = ((a0 + a1) + (a2 + a3)) + c0;
    } else if ((int)blockIdx.x >= nb + kH) {
        // grad W_out[64:][j][o] = sum_i enc[i][j] A[i][o]: 64 outputs x 4 i-slices per block
        const int e = (blockIdx.x - nb - kH) * kH + j;
        double v0 = 0.0, v1 = 0.0;
        if (e < kH * dd) {
            const int jj = e / dd, o = e - jj * dd;
            int i = q;
            for (; i + 4 < T; i += 8) {
                v0 = fma(enc_h[(size_t)i * kH + jj], A[(size_t)i * dd + o], v0);
                v1 = fma(enc_h[(size_t)(i + 4) * kH + jj], A[(size_t)(i + 4) * dd + o], v1);
            }
            if (i < T) v0 = fma(enc_h[(size_t)i * kH + jj], A[(size_t)i * dd + o], v0);
        }
        part[q][j] = v0 + v1;
        __syncthreads();
        if (q == 0 && e < kH * dd)
            grad[dm.off.w_out + (size_t)kH * dd + e] = (part[0][j] + part[1][j]) + (part[2][j] + part[3][j]);
    } else {
        const int l = blockIdx.x - nb;
        double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
        int i = q;
        for (; i + 12 < T; i += 16) {
            a0 = fma(G[(size_t)i * kH + l], enc_h[(size_t)i * kH + j], a0);
            a1 = fma(G[(size_t)(i + 4) * kH + l], enc_h[(size_t)(i + 4) * kH + j], a1);
            a2 = fma(G[(size_t)(i + 8) * kH + l], enc_h[(size_t)(i + 8) * kH + j], a2);
            a3 = fma(G[(size_t)(i + 12) * kH + l], enc_h[(size_t)(i + 12) * kH + j], a3);
        }
        for (; i < T; i += 4) a0 = fma(G[(size_t)i * kH + l], enc_h[(size_t)i * kH + j], a0);
        part[q][j] = (a0 + a1) + (a2 + a3);
        __syncthreads();
        if (q == 0) g_watt[(size_t)l * kH + j] = (part[0][j] + part[1][j]) + (part[2][j] + part[3][j]);
    }
}

// ------------------------------------------------------------------ B1a
// With A = sum_rows alpha^T du (T x dd, advantage-weighted):
//   d_enc[i, j] += sum_o A[i, o] W_out[64 + j, o]   (== sum_rows alpha^T dctx)
//   grad w_out[64 + j, o] = sum_i enc[i, j] A[i, o] (== sum_rows ctx^T du, policy.py:385)
// Blocks [0, nb) do the first (thread per d_enc element), the rest the second.
__global__ void __launch_bounds__(256) att_fin_kernel(PolicyDims dm, const double *__restrict__ P,
                                                      const double *__restrict__ enc_h, const double *__restrict__ A,
                                                      double *__restrict__ d_enc, double *__restrict__ grad, int nb) {
    const int T = dm.T, dd = dm.dd;
    const double *w2 = P + dm.off.w_out + (size_t)kH * dd;
    if ((int)blockIdx.x < nb) {
        const int e = blockIdx.x * 256 + threadIdx.x;
        if (e >= T * kH) return;
        const int i = e >> 6, j = e & 63;
        double v0 = 0.0, v1 = 0.0;
        int o = 0;
        for (; o + 2 <= dd; o += 2) {
            v0 = fma(A[(size_t)i * dd + o], w2[(size_t)j * dd + o], v0);
            v1 = fma(A[(size_t)i * dd + o + 1], w2[(size_t)j * dd + o + 1], v1);
        }
        if (o < dd) v0 = fma(A[(size_t)i * dd + o], w2[(size_t)j * dd + o], v0);
        d_enc[e] += v0 + v1;
        return;
    }
    // 32 outputs x 8 i-slices per block, fixed-order combine (deterministic)
    __shared__ double part[8][32];
    const int el = threadIdx.x & 31, sl = threadIdx.x >> 5;
    const int e = (blockIdx.x - nb) * 32 + el;
    double v0 = 0.0, v1 = 0.0;
    if (e < kH * dd) {
        const int j = e / dd, o = e - j * dd;
        int i = sl;
        for (; i + 8 < T; i += 16) {
            v0 = fma(enc_h[(size_t)i * kH + j], A[(size_t)i * dd + o], v0);
            v1 = fma(enc_h[(size_t)(i + 8) * kH + j], A[(size_t)(i + 8) * dd + o], v1);
        }
        if (i < T) v0 = fma(enc_h[(size_t)i * kH + j], A[(size_t)i * dd + o], v0);
    }
    part[sl][el] = v0 + v1;
    __syncthreads();
    if (sl == 0 && e < kH * dd) {
        double v = part[0][el];
#pragma unroll
        for (int q = 1; q < 8; q++) v += part[q][el];
        grad[dm.off.w_out + (size_t)kH * dd + e] = v;
    }
}

// ------------------------------------------------------------------ B1f
// dh_ext[r, l] += sum_j W_att[l, j] dq[r, j] ; partial w_att grad [l, j] += sum_r h[r, l] dq[r, j]
struct FinSmem {
    double watt[kH * kPad];
    double q[kFinTile * kPad];
    double h[kFinTile * kPad];
};

__global__ void __launch_bounds__(kThreads) row_fin_kernel(PolicyDims dm, const double *__restrict__ P, int rows,
                                                           int tiles_per_cta, const double *__restrict__ act_h,
                                                           const double *__restrict__ row_dq,
                                                           double *__restrict__ row_dhx, double *__restrict__ partial,
                                                           const double *__restrict__ adv, int mode) {
    extern __shared__ __align__(16) double smraw[];
    FinSmem &S = *reinterpret_cast<FinSmem *>(smraw);
    const int tid = threadIdx.x;
    const bool rows_out = mode == kFused || mode == kRowsOnly, grads_out = mode != kRowsOnly;
    const int T = dm.T;
    for (int x = tid; x < kH * kH; x += kThreads) S.watt[(x >> 6) * kPad + (x & 63)] = P[dm.off.w_att + x];
    const int rb4 = tid >> 4, lb = tid & 15;  // out micro-tile: r in {rb4+16a}, l in {lb+16b}
    double g[4][4];
#pragma unroll
    for (int a = 0; a < 4; a++)
#pragma unroll
        for (int b = 0; b < 4; b++) g[a][b] = 0.0;
    const int n_tiles = (rows + kFinTile - 1) / kFinTile;
    const int t0 = blockIdx.x * tiles_per_cta, t1 = min(n_tiles, t0 + tiles_per_cta);
    for (int tl = t0; tl < t1; tl++) {
        const int rb = tl * kFinTile;
        __syncthreads();
        for (int x = tid; x < kFinTile * kH; x += kThreads) {
            const int r = x >> 6, j = x & 63, row = rb + r;
            const bool ok = row < rows;
            S.q[r * kPad + j] = ok ? row_dq[(size_t)row * kH + j] : 0.0;
            // grads-only: dq is unscaled, fold the row's advantage into h
            const double hv = ok ? act_h[(size_t)row * kH + j] : 0.0;
            S.h[r * kPad + j] = (ok && mode == kGradsOnly) ? adv[row / T] * hv : hv;
        }
        __syncthreads();
        if (rows_out) {
            double o[4][4];
#pragma unroll
            for (int a = 0; a < 4; a++)
#pragma unroll
                for (int b = 0; b < 4; b++) o[a][b] = 0.0;
#pragma unroll 4
            for (int j = 0; j < kH; j++) {
                double qv[4], wv[4];
#pragma unroll
                for (int a = 0; a < 4; a++) qv[a] = S.q[(rb4 + 16 * a) * kPad + j];
#pragma unroll
                for (int b = 0; b < 4; b++) wv[b] = S.watt[(lb + 16 * b) * kPad + j];
#pragma unroll
                for (int a = 0; a < 4; a++)
#pragma unroll
                    for (int b = 0; b < 4; b++) o[a][b] = fma(qv[a], wv[b], o[a][b]);
            }
#pragma unroll
            for (int a = 0; a < 4; a++) {
                const int row = rb + rb4 + 16 * a;
                if (row < rows)
#pragma unroll
                    for (int b = 0; b < 4; b++) row_dhx[(size_t)row * kH + lb + 16 * b] += o[a][b];
            }
        }
        // grad: l in {rb4 + 16a} (reuse mapping), j in {lb + 16b}
        if (!grads_out) continue;
#pragma unroll 4
        for (int r = 0; r < kFinTile; r++) {
            double hv[4], qv[4];
#pragma unroll
            for (int a = 0; a < 4; a++) hv[a] = S.h[r * kPad + rb4 + 16 * a];
#pragma unroll
            for (int b = 0; b < 4; b++) qv[b] = S.q[r * kPad + lb + 16 * b];
#pragma unroll
            for (int a = 0; a < 4; a++)
#pragma unroll
                for (int b = 0; b < 4; b++) g[a][b] = fma(hv[a], qv[b], g[a][b]);
        }
    }
    if (!grads_out) return;
#pragma unroll
    for (int a = 0; a < 4; a++)
#pragma unroll
        for (int b = 0; b < 4; b++)
            partial[(size_t)blockIdx.x * kH * kH + (rb4 + 16 * a) * kH + lb + 16 * b] = g[a][b];
}

// ------------------------------------------------------------------ B2 / B4
// Sequential LSTM backward (pkg/policy.py:236-253) for M (<= 4) sequences per
// CTA, 256 threads (8 warps: fewer barrier participants than 16 measured
// faster).  Lane j of warp w keeps W_h[8w .. 8w+7, j + 32q] (q < 8) in
// registers; dh_prev = W_h da by lane-parallel partial sums and a
// reduce-scatter butterfly.  One elementwise slot (m, u) per thread.  The next
// step's gate activations / cells / incoming dh are prefetched into registers
// while the current step's mat-vec runs.  In place: gate activations become da.
constexpr int kLstmThreads = 256;
constexpr int kMaxSeqPerCta = kLstmThreads / 64;   // one elementwise slot (sample, unit) per thread
constexpr int kRpw = kH / (kLstmThreads / 32);     // W_h rows per warp in the mat-vec
__device__ int g_lstm_dbg = 0;            // debug-only phase clocks of lstm_bwd (block 0, thread 0)
static bool g_lstm_clocks_on = false;      // host side: launch the CLK instantiations
__device__ long long g_lstm_clk[2][4];    // [M == 1 ? 0 : 1][phase]
// Mat-vec mapping: lane j of warp w owns gate columns {j + 32q} (q < 8) of
// W_h rows 4w..4w+3 (32 weights in registers).  Every lane reads a DIFFERENT
// da value (8 conflict-free LDS.64 per sample per thread: 16 shared-memory
// wavefronts per warp, 4x fewer than a part-per-row layout whose lanes re-read
// the same slices), then a reduce-scatter butterfly (6 shuffles) leaves row
// sums on lanes 0, 8, 16, 24.
inline size_t lstm_bwd_smem(int M) { return sizeof(double) * (size_t)M * (2 * kH + kG); }

// CLK: debug phase clocks compiled in (disabled instrumentation still costs
// issue slots on this latency-bound chain), launched only while enabled
template <int MT, bool CLK = false>
__global__ void __launch_bounds__(kLstmThreads, 1) lstm_bwd_kernel(
    int T, int n_seq, int M, const double *__restrict__ Wh /* [64 x 256] row-major, ld 256 */,
    double *__restrict__ gates /* [seq][T][256] in: i,f,o,g  out: da */, const double *__restrict__ cst /* [seq][T][64] */,
    const double *__restrict__ c_init /* [64] c before step 0 */, const double *__restrict__ dh_ext /* [seq][T][64] */,
    const double *__restrict__ dh_in /* [seq][64] or NULL */, const double *__restrict__ dc_in,
    double *__restrict__ dh_out /* [seq][64] */, double *__restrict__ dc_out,
    const double *__restrict__ gates_in /* activations read (== gates: in place) */,
    const double *__restrict__ sum_dh /* M == 1, non-NULL: dh_in = sum_r sum_w[r] sum_dh[r], dc_in likewise */,
    const double *__restrict__ sum_dc, const double *__restrict__ sum_w, int sum_rows,
    int *__restrict__ colexp /* [256] or NULL: max biased exponent of |da| per gate column */) {
    extern __shared__ __align__(16) double sm[];
    double *s_dh = sm;                   // [M][64]
    double *s_dc = s_dh + M * kH;        // [M][64]
    double *s_da = s_dc + M * kH;        // [M][256] gate columns (i, f, o, g blocks of 64)
    const int tid = threadIdx.x;
    const int q0 = blockIdx.x * M;
    const int Mb = min(M, n_seq - q0);
    const int lane = tid & 31, wrow = (tid >> 5) * kRpw;  // rows wrow.., columns lane + 32q
    double w[kRpw][8];
#pragma unroll
    for (int rr = 0; rr < kRpw; rr++)
#pragma unroll
        for (int q = 0; q < 8; q++) w[rr][q] = Wh[(size_t)(wrow + rr) * kG + lane + 32 * q];
    if (sum_dh) {
        // encoder: the decoders' step-0 state gradients, advantage-weighted and
        // summed over the samples: thread (u, which = dh|dc, slice of 2), fixed-
        // order combine; scratch in s_da (256 doubles, free until the first step)
        static_assert(kLstmThreads == 4 * kH, "the prologue sum maps 256 threads to (u, which, slice)");
        double *part = s_da;  // [which][slice][64]
        const int u = tid & 63, sl = (tid >> 6) & 1, which = tid >> 7;
        const double *src = which ? sum_dc : sum_dh;
        double a0 = 0.0, a1 = 0.0;
        int r = sl;
        for (; r + 2 < sum_rows; r += 4) {
            a0 = fma(sum_w ? sum_w[r] : 1.0, src[(size_t)r * kH + u], a0);
            a1 = fma(sum_w ? sum_w[r + 2] : 1.0, src[(size_t)(r + 2) * kH + u], a1);
        }
        if (r < sum_rows) a0 = fma(sum_w ? sum_w[r] : 1.0, src[(size_t)r * kH + u], a0);
        part[(which * 2 + sl) * kH + u] = a0 + a1;
        __syncthreads();
        if (tid < kH) {
            s_dh[tid] = part[tid] + part[kH + tid];
            s_dc[tid] = part[2 * kH + tid] + part[3 * kH + tid];
        }
    } else {
        for (int x = tid; x < Mb * kH; x += kLstmThreads) {
            const int m = x >> 6, u = x & 63;
            s_dh[x] = dh_in ? dh_in[(size_t)(q0 + m) * kH + u] : 0.0;
            s_dc[x] = dc_in ? dc_in[(size_t)(q0 + m) * kH + u] : 0.0;
        }
    }
    // elementwise slot of this thread: x = tid (M <= 8 -> Mb*64 <= 512)
    const int x = tid, xm = x >> 6, xu = x & 63;
    const bool live = x < Mb * kH;
    // two-deep register prefetch (rotating cur <- nxt): step t-1's operands were
    // issued a whole step earlier, t-2's are issued while step t runs; tanh(c)
    // of the coming step is evaluated inside the mat-vec section, where its
    // latency overlaps the FMA chains instead of the elementwise critical path
    struct Ops {
        double i, f, o, g, c, cp, dx;
    };
    Ops cur{0, 0, 0, 0, 0, 0, 0}, nxt{0, 0, 0, 0, 0, 0, 0};
    auto load = [&](int t, Ops &d) {
        if (live && t >= 0) {
            const size_t row = (size_t)(q0 + xm) * T + t;
            const double *g = gates_in + row * kG;
            d.i = g[xu];
            d.f = g[kH + xu];
            d.o = g[2 * kH + xu];
            d.g = g[3 * kH + xu];
            d.c = cst[row * kH + xu];
            d.cp = t > 0 ? cst[(row - 1) * kH + xu] : c_init[xu];
            d.dx = dh_ext[row * kH + xu];
        }
    };
    load(T - 1, cur);
    load(T - 2, nxt);
    double tc = fm_gate_act(cur.c, true);  // tanh (branch-free, fastmath.cuh)

    const bool clk_on = CLK && blockIdx.x == 0 && tid == 0;
    const int ci = M == 1 ? 0 : 1;
    long long clk_last = clk_on ? clock64() : 0;
    long long clk_acc[4] = {0, 0, 0, 0};  // in registers; one global write at the end
#define DP_LPHASE(i)                                   \
    if (clk_on) {                                      \
        const long long now_ = clock64();              \
        clk_acc[i] += now_ - clk_last;                 \
        clk_last = now_;                               \
    }
    __syncthreads();
    // this slot's da row in the gates array (in place), walked backwards
    double *grow = gates + ((size_t)(q0 + (live ? xm : 0)) * T + (T - 1)) * kG + xu;
    // running max exponent of |da| per gate column (the tensor-core weight
    // gradient's fixed-point scales, wgrad_tc.cu); integer max of the
    // exponent fields, off the elementwise chain
    int ex_i = 0, ex_f = 0, ex_o = 0, ex_g = 0;
    auto expo = [](double v) { return (__double2hiint(v) >> 20) & 0x7FF; };
    for (int t = T - 1; t >= 0; t--, grow -= kG) {
        double da_i = 0.0, da_f = 0.0, da_o = 0.0, da_g = 0.0;
        if (live) {
            const double iv = cur.i, fv = cur.f, ov = cur.o, gv = cur.g, cp = cur.cp;
            const double dh = s_dh[x] + cur.dx;
            const double d_o = dh * tc;
            const double dcv = s_dc[x] + dh * ov * (1.0 - tc * tc);
            const double di = dcv * gv;
            const double dg = dcv * iv;
            const double df = dcv * cp;
            s_dc[x] = dcv * fv;
            da_i = di * iv * (1.0 - iv);
            da_f = df * fv * (1.0 - fv);
            da_o = d_o * ov * (1.0 - ov);
            da_g = dg * (1.0 - gv * gv);
            double *sd = s_da + xm * kG + xu;
            sd[0] = da_i;
            sd[kH] = da_f;
            sd[2 * kH] = da_o;
            sd[3 * kH] = da_g;
        }
        cur = nxt;
        load(t - 2, nxt);  // lands during this and the next step's barrier + mat-vec
        DP_LPHASE(0);
        __syncthreads();
        DP_LPHASE(1);
        if (live) {
            // the global da row after the barrier: off the elementwise chain
            grow[0] = da_i;
            grow[kH] = da_f;
            grow[2 * kH] = da_o;
            grow[3 * kH] = da_g;
            ex_i = max(ex_i, expo(da_i));
            ex_f = max(ex_f, expo(da_f));
            ex_o = max(ex_o, expo(da_o));
            ex_g = max(ex_g, expo(da_g));
        }
        if (live) tc = fm_gate_act(cur.c, true);  // tanh; independent of the mat-vec below: the chains interleave
        // per sample: partial row sums over this lane's 8 columns, then a
        // reduce-scatter butterfly: each xor level halves the rows a lane
        // carries until one is left, the remaining levels sum (fixed tree)
#pragma unroll
        for (int m = 0; m < MT; m++) {
            if (m >= Mb) break;
            double p[kRpw];
            {
                double dv[8];
#pragma unroll
                for (int q = 0; q < 8; q++) dv[q] = s_da[m * kG + lane + 32 * q];
#pragma unroll
                for (int rr = 0; rr < kRpw; rr++) {
                    double a0 = 0.0, a1 = 0.0;
#pragma unroll
                    for (int q = 0; q < 8; q += 2) {
                        a0 = fma(w[rr][q], dv[q], a0);
                        a1 = fma(w[rr][q + 1], dv[q + 1], a1);
                    }
                    p[rr] = a0 + a1;
                }
            }
            int rbase = 0;
#pragma unroll
            for (int o = 16, cnt = kRpw; o >= 1; o >>= 1) {
                const bool hi = lane & o;
                if (cnt > 1) {
                    const int half = cnt / 2;
#pragma unroll
                    for (int i2 = 0; i2 < kRpw / 2; i2++)
                        if (i2 < half) {
                            const double send = hi ? p[i2] : p[i2 + half];
                            const double keep = hi ? p[i2 + half] : p[i2];
                            p[i2] = keep + __shfl_xor_sync(0xffffffffu, send, o);
                        }
                    rbase += hi ? half : 0;
                    cnt = half;
                } else {
                    p[0] += __shfl_xor_sync(0xffffffffu, p[0], o);
                }
            }
            if ((lane & (32 / kRpw - 1)) == 0) s_dh[m * kH + wrow + rbase] = p[0];
        }
        DP_LPHASE(2);
        __syncthreads();
        DP_LPHASE(3);
    }
#undef DP_LPHASE
    if (clk_on)
#pragma unroll
        for (int i = 0; i < 4; i++) g_lstm_clk[ci][i] += clk_acc[i];
    if (colexp && live) {
        atomicMax(colexp + xu, ex_i);
        atomicMax(colexp + kH + xu, ex_f);
        atomicMax(colexp + 2 * kH + xu, ex_o);
        atomicMax(colexp + 3 * kH + xu, ex_g);
    }
    for (int y = tid; y < Mb * kH; y += kLstmThreads) {
        const int m = y >> 6, u = y & 63;
        dh_out[(size_t)(q0 + m) * kH + u] = s_dh[y];
        dc_out[(size_t)(q0 + m) * kH + u] = s_dc[y];
    }
}

const void *lstm_bwd_fn(int M) {
    static_assert(kMaxSeqPerCta == 4, "lstm_bwd_fn instantiates MT <= 4");
    if (g_lstm_clocks_on)
        return M <= 1 ? (const void *)lstm_bwd_kernel<1, true>
               : M <= 2 ? (const void *)lstm_bwd_kernel<2, true>
                        : (const void *)lstm_bwd_kernel<4, true>;
    return M <= 1 ? (const void *)lstm_bwd_kernel<1>
           : M <= 2 ? (const void *)lstm_bwd_kernel<2>
                    : (const void *)lstm_bwd_kernel<4>;
}

// ------------------------------------------------------------------ B3
// partial per CTA: [Hg (64 x 256) | DAsum ((D+1) x 256)]
// Hg = (adv o H_prev)^T DA and DAsum[p] = sum over rows whose previous choice
// is p of adv * da, on the fp64 tensor cores (DMMA m8n8k4): warp w owns
// m-tiles 2(w&3), 2(w&3)+1 (rows l of Hg) x n-tiles 16(w>>2) .. +16 (columns
// j); for D+1 <= 8 DAsum is one more m-tile whose A fragment is the one-hot
// of the row's previous choice times its advantage (warp w: n-tiles
// 16(w>>2) + 4(w&3) .. +4, reusing the B fragments it already loaded).
// Tiles of 32 rows (h_prev, da, advantages, choice bytes) stream through a
// cp.async double buffer with row strides == 8 (mod 32) words (conflict-free
// fragment loads); the advantage scales the A fragments in registers.
constexpr int kWgHLd = kH + 4, kWgDLd = kG + 4;
__global__ void __launch_bounds__(kThreads, 1) dec_wgrad_kernel(PolicyDims dm, int rows, int tiles_per_cta,
                                                                const double *__restrict__ act_h,
                                                                const double *__restrict__ enc_h,
                                                                const uint8_t *__restrict__ choice,
                                                                const double *__restrict__ da,
                                                                double *__restrict__ partial,
                                                                const double *__restrict__ adv) {
    extern __shared__ __align__(16) double sm[];
    double *s_h = sm;                              // [2][kTile][kWgHLd]   (cp.async double buffer)
    double *s_da = s_h + 2 * kTile * kWgHLd;       // [2][kTile][kWgDLd]
    double *s_dasum = s_da + 2 * kTile * kWgDLd;   // [(D+1)][256] (D+1 > 8 only)
    __shared__ double s_w[2][kTile];               // per-row advantage (1 when already scaled)
    __shared__ __align__(8) uint8_t s_ch[2][kTile + 8];  // choices of rows rb-8 .. rb+31
    const int tid = threadIdx.x, lane = tid & 31, wp = tid >> 5, g = lane >> 2, t = lane & 3;
    const int T = dm.T, D = dm.D;
    const bool oh = D + 1 <= 8;
    const int mt0 = (wp & 3) * 2, nt0 = (wp >> 2) * 16, no0 = (wp & 3) * 4;
    double acc[2][16][2], acc_oh[4][2];
#pragma unroll
    for (int a = 0; a < 2; a++)
#pragma unroll
        for (int n = 0; n < 16; n++) acc[a][n][0] = acc[a][n][1] = 0.0;
#pragma unroll
    for (int n = 0; n < 4; n++) acc_oh[n][0] = acc_oh[n][1] = 0.0;
    if (!oh)
        for (int p = 0; p <= D; p++) s_dasum[p * kG + tid] = 0.0;
    const int n_tiles = (rows + kTile - 1) / kTile;
    const int t0 = blockIdx.x * tiles_per_cta, t1 = min(n_tiles, t0 + tiles_per_cta);
    // async copy of tile tl into buffer b (cp.async, zero-fill past the end)
    auto stage = [&](int tl, int b) {
        const int rb = tl * kTile;
        double *h = s_h + b * kTile * kWgHLd, *d = s_da + b * kTile * kWgDLd;
        for (int x = tid * 2; x < kTile * kH; x += kThreads * 2) {
            const int r = x >> 6, l = x & 63, row = rb + r;
            const bool ok = row < rows;
            const double *src = enc_h + (size_t)(T - 1) * kH + l;
            if (ok && row % T > 0) src = act_h + (size_t)(row - 1) * kH + l;
            cp_async16(h + r * kWgHLd + l, src, ok);
        }
        for (int x = tid * 2; x < kTile * kG; x += kThreads * 2) {
            const int r = x >> 8, c = x & 255, row = rb + r;
            cp_async16(d + r * kWgDLd + c, da + (size_t)rb * kG + (row < rows ? x : 0), row < rows);
        }
        if (tid < kTile) {
            const int row = rb + tid;
            const bool ok = row < rows;
            if (adv) cp_async8(&s_w[b][tid], adv + (ok ? row / T : 0), ok);
            else s_w[b][tid] = ok ? 1.0 : 0.0;
        } else if (tid < kTile + (kTile + 8) / 8) {
            // 8-byte words of the choice bytes of rows rb-8 .. rb+31 (rb is 32-aligned)
            const int q = tid - kTile, row = rb - 8 + 8 * q;
            if (row >= 0 && row + 8 <= rows) {
                cp_async8(&s_ch[b][8 * q], choice + row, true);
            } else {
                for (int e = 0; e < 8; e++) s_ch[b][8 * q + e] = row + e >= 0 && row + e < rows ? choice[row + e] : 0;
            }
        }
        cp_async_commit();
    };
    if (t0 < t1) stage(t0, 0);
    for (int tl = t0; tl < t1; tl++) {
        const int b = (tl - t0) & 1;
        const int rb = tl * kTile;
        if (tl + 1 < t1) {
            stage(tl + 1, b ^ 1);  // next tile in flight while this one is used
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncthreads();
        const double *h = s_h + b * kTile * kWgHLd;
        const double *d = s_da + b * kTile * kWgDLd;
#pragma unroll 2
        for (int ks = 0; ks < kTile / 4; ks++) {
            const int r = ks * 4 + t, row = rb + r;
            const double wr = s_w[b][r];
            const double a0 = h[r * kWgHLd + mt0 * 8 + g] * wr, a1 = h[r * kWgHLd + (mt0 + 1) * 8 + g] * wr;
            // one-hot A fragment: row r's previous choice (D at the sequence start)
            const int pv = row % T > 0 ? (int)s_ch[b][r + 7] : D;
            const double ao = pv == g ? wr : 0.0;
#pragma unroll
            for (int n = 0; n < 16; n++) {
                const double bb = d[r * kWgDLd + (nt0 + n) * 8 + g];
                dmma884(acc[0][n], a0, bb);
                dmma884(acc[1][n], a1, bb);
            }
            if (oh)
#pragma unroll
                for (int n = 0; n < 4; n++) dmma884(acc_oh[n], ao, d[r * kWgDLd + (nt0 + no0 + n) * 8 + g]);
        }
        if (!oh) {
            const int nr = min(kTile, rows - rb);
            for (int r = 0; r < nr; r++) {
                const int row = rb + r;
                const int pv = row % T > 0 ? (int)s_ch[b][r + 7] : D;
                s_dasum[pv * kG + tid] += s_w[b][r] * d[r * kWgDLd + tid];
            }
        }
        __syncthreads();  // buffer b is re-staged by the next iteration
    }
    const size_t base = (size_t)blockIdx.x * (kH + D + 1) * kG;
#pragma unroll
    for (int a = 0; a < 2; a++)
#pragma unroll
        for (int n = 0; n < 16; n++)
            *reinterpret_cast<double2 *>(partial + base + (size_t)((mt0 + a) * 8 + g) * kG + (nt0 + n) * 8 + 2 * t) =
                make_double2(acc[a][n][0], acc[a][n][1]);
    if (oh) {
        if (g <= D)
#pragma unroll
            for (int n = 0; n < 4; n++)
                *reinterpret_cast<double2 *>(partial + base + (size_t)(kH + g) * kG + (nt0 + no0 + n) * 8 + 2 * t) =
                    make_double2(acc_oh[n][0], acc_oh[n][1]);
    } else {
        for (int p = 0; p <= D; p++) partial[base + (size_t)(kH + p) * kG + tid] = s_dasum[p * kG + tid];
    }
}

// ------------------------------------------------------------------ reductions
// dst[e] (+)= sum_c (w[c / tps] *) src[c * stride + e] for up to 4 (src,
// stride, n, dst) segments in one launch (block ranges b0[i] .. b0[i+1]).
// Block = 32 elements x 16 c-slices, 4 loads in flight per thread; the slice
// sums combine in a fixed order -> deterministic (the partials are latency-,
// not bandwidth-bound).  w != NULL: advantage-weighted per-sample partials.
constexpr int kRedSl = 16;
struct RedSegs {
    const double *src[4];
    double *dst[4];
    size_t stride[4];
    int n[4];
    int b0[5];
    int count;
};
__global__ void __launch_bounds__(32 * kRedSl) reduce_multi_kernel(RedSegs sg, int n_cta, int accumulate,
                                                                   const double *__restrict__ w, int tps) {
    __shared__ double part[kRedSl][32];
    const int el = threadIdx.x & 31, s = threadIdx.x >> 5;
    int i = 0;
    while (i + 1 < sg.count && (int)blockIdx.x >= sg.b0[i + 1]) i++;
    const double *src = sg.src[i];
    const size_t stride = sg.stride[i];
    const int n = sg.n[i];
    const int e = (blockIdx.x - sg.b0[i]) * 32 + el;
    double v0 = 0.0, v1 = 0.0, v2 = 0.0, v3 = 0.0;
    if (e < n) {
        int c = s;
        for (; c + 3 * kRedSl < n_cta; c += 4 * kRedSl) {
            const double x0 = src[(size_t)c * stride + e], x1 = src[(size_t)(c + kRedSl) * stride + e];
            const double x2 = src[(size_t)(c + 2 * kRedSl) * stride + e];
            const double x3 = src[(size_t)(c + 3 * kRedSl) * stride + e];
            if (w) {
                v0 = fma(w[c / tps], x0, v0);
                v1 = fma(w[(c + kRedSl) / tps], x1, v1);
                v2 = fma(w[(c + 2 * kRedSl) / tps], x2, v2);
                v3 = fma(w[(c + 3 * kRedSl) / tps], x3, v3);
            } else {
                v0 += x0;
                v1 += x1;
                v2 += x2;
                v3 += x3;
            }
        }
        for (; c < n_cta; c += kRedSl) {
            const double x = src[(size_t)c * stride + e];
            v0 = w ? fma(w[c / tps], x, v0) : v0 + x;
        }
    }
    part[s][el] = (v0 + v1) + (v2 + v3);
    __syncthreads();
    if (s == 0 && e < n) {
        double v = part[0][el];
#pragma unroll
        for (int q = 1; q < kRedSl; q++) v += part[q][el];
        double *dst = sg.dst[i];
        dst[e] = accumulate ? dst[e] + v : v;
    }
}

struct RedBuilder {
    RedSegs sg{};
    int blocks = 0;
    void add(const double *src, size_t stride, int n, double *dst) {
        const int i = sg.count++;
        sg.src[i] = src;
        sg.dst[i] = dst;
        sg.stride[i] = stride;
        sg.n[i] = n;
        sg.b0[i] = blocks;
        blocks += (n + 31) / 32;
        sg.b0[i + 1] = blocks;
    }
    void launch(int n_cta, int accumulate, cudaStream_t st, const double *w = nullptr, int tps = 1) {
        if (blocks) reduce_multi_kernel<<<blocks, 32 * kRedSl, 0, st>>>(sg, n_cta, accumulate, w, tps);
    }
};

inline void launch_reduce(const double *src, int n_cta, size_t stride, int n, double *dst, int accumulate,
                          cudaStream_t st) {
    RedBuilder rb;
    rb.add(src, stride, n, dst);
    rb.launch(n_cta, accumulate, st);
}

// B3 finalize: b_dec = sum_p DAsum[p]; w_dec[:dd] = sum_p dev_table[p] x DAsum[p];
// dev_table[p] += W_dec[:dd] . DAsum[p]
// Block 0: thread per gate column (b_dec, w_dec[:dd]); blocks >= 1: one warp
// per dev_table output (p, i), lanes split the 256 gates, fixed butterfly.
__global__ void __launch_bounds__(kG) dec_finalize_kernel(PolicyDims dm, const double *__restrict__ P,
                                                          const double *__restrict__ dasum,
                                                          double *__restrict__ grad) {
    const int tid = threadIdx.x;
    const int D = dm.D, dd = dm.dd;
    if (blockIdx.x == 0) {
        double b = 0.0;
        for (int p = 0; p <= D; p++) b += dasum[p * kG + tid];
        grad[dm.off.b_dec + tid] = b;
        for (int i = 0; i < dd; i++) {
            double v = 0.0;
            for (int p = 0; p <= D; p++) v = fma(P[dm.off.dev_table + p * dd + i], dasum[p * kG + tid], v);
            grad[dm.off.w_dec + (size_t)i * kG + tid] = v;
        }
        return;
    }
    const int x = (blockIdx.x - 1) * (kG / 32) + (tid >> 5), lane = tid & 31;
    if (x >= (D + 1) * dd) return;
    const int p = x / dd, i = x - p * dd;
    double v = 0.0;
#pragma unroll
    for (int q = 0; q < kG / 32; q++) {
        const int j = lane + 32 * q;
        v = fma(P[dm.off.w_dec + (size_t)i * kG + j], dasum[p * kG + j], v);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) grad[dm.off.dev_table + x] += v;
}

// B5: w_enc / b_enc grads (contraction over T) and the type-embedding scatter.
// enc_wgrad: block = 4 rows r of [X | h_prev] (or b_enc) x 256 gate columns;
// the 4 input rows are staged in shared memory, da_enc streams through a
// cp.async double buffer of 16-step chunks (bulk loads instead of one L2
// latency per step and thread).
constexpr int kWgRows = 4, kWgChunk = 16;
inline size_t enc_wgrad_smem(int T) { return sizeof(double) * ((size_t)kWgRows * T + 2 * kWgChunk * kG); }
__global__ void __launch_bounds__(kG) enc_wgrad_kernel(PolicyDims dm, const double *__restrict__ X,
                                                       const double *__restrict__ enc_h,
                                                       const double *__restrict__ da_enc, double *__restrict__ grad) {
    extern __shared__ __align__(16) double xs[];  // [kWgRows][T], then [2][kWgChunk][256]
    const int j = threadIdx.x;
    const int T = dm.T, F = dm.F;
    const int r0 = blockIdx.x * kWgRows;
    double *dab = xs + kWgRows * T;
    const int n_chunks = (T + kWgChunk - 1) / kWgChunk;
    auto stage = [&](int c, int b) {
        double *dst = dab + b * kWgChunk * kG;
        const double *src = da_enc + (size_t)c * kWgChunk * kG;
        for (int x = j * 2; x < kWgChunk * kG; x += kG * 2) {
            const bool ok = c * kWgChunk + x / kG < T;
            cp_async16(dst + x, ok ? src + x : da_enc, ok);
        }
        cp_async_commit();
    };
    stage(0, 0);
    for (int x = j; x < kWgRows * T; x += kG) {
        const int a = x / T, t = x - a * T, r = r0 + a;
        double v = 0.0;
        if (r < F) v = X[(size_t)t * F + r];
        else if (r < F + kH) v = t > 0 ? enc_h[(size_t)(t - 1) * kH + (r - F)] : 0.0;
        else if (r == F + kH) v = 1.0;  // b_enc row
        xs[x] = v;
    }
    double acc[kWgRows][2];
#pragma unroll
    for (int a = 0; a < kWgRows; a++) acc[a][0] = acc[a][1] = 0.0;
    for (int c = 0; c < n_chunks; c++) {
        const int b = c & 1;
        if (c + 1 < n_chunks) {
            stage(c + 1, b ^ 1);
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncthreads();
        const double *d = dab + b * kWgChunk * kG;
        const int tb = c * kWgChunk, nt = min(kWgChunk, T - tb);
        if (nt == kWgChunk) {
#pragma unroll 8
            for (int tt = 0; tt < kWgChunk; tt += 2) {
                const double d0 = d[tt * kG + j], d1 = d[(tt + 1) * kG + j];
#pragma unroll
                for (int a = 0; a < kWgRows; a++) {
                    acc[a][0] = fma(xs[a * T + tb + tt], d0, acc[a][0]);
                    acc[a][1] = fma(xs[a * T + tb + tt + 1], d1, acc[a][1]);
                }
            }
        } else {
            for (int tt = 0; tt < nt; tt++) {
                const double d0 = d[tt * kG + j];
#pragma unroll
                for (int a = 0; a < kWgRows; a++) acc[a][0] = fma(xs[a * T + tb + tt], d0, acc[a][0]);
            }
        }
        __syncthreads();  // buffer b is re-staged two chunks on
    }
#pragma unroll
    for (int a = 0; a < kWgRows; a++) {
        const int r = r0 + a;
        if (r < F + kH) grad[dm.off.w_enc + (size_t)r * kG + j] = acc[a][0] + acc[a][1];
        else if (r == F + kH) grad[dm.off.b_enc + j] = acc[a][0] + acc[a][1];
    }
}

// dx_t[f] = W_enc[f, :] . da_enc[t]   (f < type_dim): block per t.  Per 32-wide f
// chunk every lane forms its 32 products (loads issued together), a
// reduce-scatter butterfly (31 shuffles) leaves f = f0 + lane's warp sum in
// lane f - f0, and the 8 warp sums combine in a fixed order.
__global__ void __launch_bounds__(kG) enc_dx_kernel(PolicyDims dm, const double *__restrict__ P,
                                                    const double *__restrict__ da_enc, double *__restrict__ dx) {
    __shared__ double part[kG / 32][32];
    const int t = blockIdx.x, j = threadIdx.x, lane = j & 31, w = j >> 5;
    const double d = da_enc[(size_t)t * kG + j];
    for (int f0 = 0; f0 < dm.td; f0 += 32) {
        double v[32];
#pragma unroll
        for (int q = 0; q < 32; q++) v[q] = f0 + q < dm.td ? P[dm.off.w_enc + (size_t)(f0 + q) * kG + j] * d : 0.0;
#pragma unroll
        for (int lv = 0; lv < 5; lv++) {
            const int o = 16 >> lv, half = 16 >> lv;  // values carried: 2 * half
            const bool hi = lane & o;
#pragma unroll
            for (int i = 0; i < half; i++) {
                const double send = hi ? v[i] : v[i + half];
                const double keep = hi ? v[i + half] : v[i];
                v[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
            }
        }
        part[w][lane] = v[0];
        __syncthreads();
        if (w == 0 && f0 + lane < dm.td) {
            double s = part[0][lane];
#pragma unroll
            for (int q = 1; q < kG / 32; q++) s += part[q][lane];
            dx[(size_t)t * dm.td + f0 + lane] = s;
        }
        __syncthreads();
    }
}

// np.add.at(type_table, idx_t, dx_t / len(idx_t)) in (t, position) order
// (pkg/policy.py:405-407).  Block per vocabulary row v: its occurrences' terms
// dx[t][f] / len(idx_t) are staged in shared memory in chunks (all loads in
// flight at once), then thread f adds them in occurrence order — the
// reference's order.
constexpr int kScatterVals = 4096;
__global__ void __launch_bounds__(256) type_scatter_kernel(PolicyDims dm, const int32_t *__restrict__ occ_off,
                                                           const int32_t *__restrict__ occ_t,
                                                           const int32_t *__restrict__ type_off,
                                                           const double *__restrict__ dx, double *__restrict__ grad) {
    __shared__ double vals[kScatterVals];
    const int v = blockIdx.x, tid = threadIdx.x, td = dm.td;
    const int o0 = occ_off[v], o1 = occ_off[v + 1];
    const int per = kScatterVals / td;  // occurrences per chunk
    double s = 0.0;
    for (int c0 = o0; c0 < o1; c0 += per) {
        const int nc = min(per, o1 - c0);
        for (int x = tid; x < nc * td; x += blockDim.x) {
            const int o = c0 + x / td, f = x - (x / td) * td;
            const int t = occ_t[o];
            vals[x] = dx[(size_t)t * td + f] / (double)(type_off[t + 1] - type_off[t]);
        }
        __syncthreads();
        if (tid < td)
#pragma unroll 8
            for (int i = 0; i < nc; i++) s = s + vals[i * td + tid];
        __syncthreads();
    }
    if (tid < td) grad[dm.off.type_table + (size_t)v * td + tid] = s;
}

int n_cta_for(int units, int min_units) {
    int n = ceil_div(units, min_units);
    if (n > 2 * kNumSMs) n = 2 * kNumSMs;
    return n < 1 ? 1 : n;
}

}  // namespace
}  // namespace dp

using namespace dp;

// Debug: LSTM-backward phase clocks [encoder (M=1) / decoder (M>1)][elementwise,
// barrier 1, tanh + mat-vec, barrier 2] into h_out[8]; read + reset.
extern "C" int dp_debug_lstm_clocks(int32_t enable, int64_t *h_out) {
    DP_ENTRY();
    const int on = enable ? 1 : 0;
    DP_CUDA_TRY(cudaMemcpyToSymbol(g_lstm_dbg, &on, sizeof(int)));
    g_lstm_clocks_on = on != 0;
    if (h_out) DP_CUDA_TRY(cudaMemcpyFromSymbol(h_out, g_lstm_clk, sizeof(long long) * 8));
    long long z[8] = {0};
    DP_CUDA_TRY(cudaMemcpyToSymbol(g_lstm_clk, z, sizeof(z)));
    return DP_OK;
}

extern "C" int dp_debug_att_clocks(int32_t enable, int64_t *h_out) {
    DP_ENTRY();
    const int on = enable ? 1 : 0;
    DP_CUDA_TRY(cudaMemcpyToSymbol(g_att_dbg, &on, sizeof(int)));
    if (h_out) DP_CUDA_TRY(cudaMemcpyFromSymbol(h_out, g_att_clk, sizeof(long long) * 8));
    long long z[8] = {0};
    DP_CUDA_TRY(cudaMemcpyToSymbol(g_att_clk, z, sizeof(z)));
    return DP_OK;
}

size_t dp_backward_partial_elems(const dp_policy *p) {
    const PolicyDims &dm = p->dims;
    const size_t ncta = 2 * kNumSMs;
    size_t a = ncta * (size_t)(dm.D + dm.D * dm.dd + 2 * kH * dm.dd);
    size_t b = ncta * (size_t)dm.T * kH;
    size_t c = ncta * (size_t)kH * kH;
    size_t d = ncta * (size_t)(kH + dm.D + 1) * kG;
    size_t e = ncta * adv_grads_partial(dm);
    size_t m = a > b ? a : b;
    m = m > e ? m : e;
    m = m > c ? m : c;
    m = m > d ? m : d;
    return m + (size_t)dm.T * dm.td + 4 * kH;  // + dx scratch + (dh, dc) sums + encoder (dh, dc) sink
}

namespace {

struct Grid {
    int n_used, per;
};
Grid tiles_grid(int rows, int tile) {
    const int n_tiles = ceil_div(rows, tile);
    const int n = n_cta_for(n_tiles, 2);
    const int per = ceil_div(n_tiles, n);
    return {ceil_div(n_tiles, per), per};
}

// one CTA per SM, each streaming a contiguous run of tiles through its
// cp.async pipeline
Grid persist_grid(int rows, int tile) {
    const int n_tiles = ceil_div(rows, tile);
    const int n = n_tiles < kNumSMs ? n_tiles : kNumSMs;
    const int per = ceil_div(n_tiles, n);
    return {ceil_div(n_tiles, per), per};
}

Grid att_grid(int K, int T, bool split) {
    // one wave: att_bwd holds ~220 KB of shared memory (1 CTA per SM).  The
    // split backward's rows pass leaves kSimSMs SMs free (it runs concurrently
    // with the placement simulator: small latency-bound CTAs that cannot
    // co-reside with an att_bwd CTA) and, when a CTA gets at least one whole
    // sample, rounds its tile range to whole samples (per-sample partials).
    // The fused pass runs after scoring, takes every SM and accumulates per CTA.
    constexpr int kSimSMs = 20;
    const int tps = (T + kAttTile - 1) / kAttTile;
    const int n_tiles = K * tps;
    const int n_sm = split ? kNumSMs - kSimSMs : kNumSMs;
    const int n = n_tiles < n_sm ? n_tiles : n_sm;
    int per = ceil_div(n_tiles, n);
    if (split && per >= tps) per = ceil_div(per, tps) * tps;
    return {ceil_div(n_tiles, per), per};
}

// Whether the rows pass's attention backward forms row_prep's per-row outputs itself
// (GM DMMA kernel: act_e stored and per-tile partials allocated, not the tcgen05 variant).
bool att_prep_merged(const dp_policy *p) {
    return p->act_e && p->tile_part && !(dp_tensor_core_mode() == 6 && att_bwd_tc_ok(p->dims));
}

int launch_att(dp_policy *p, const double *params, const Grid &g, size_t smem, int rows, double *tile_part,
               double *tile_partA, cudaStream_t st, int prep = 0) {
    const PolicyDims &dm = p->dims;
    const int tps = (dm.T + kAttTile - 1) / kAttTile;
    const int per_sample = tile_part && g.per % tps == 0 ? 1 : 0;
    p->att_per_sample = per_sample;
    p->att_gmode = p->act_e && tile_part ? 1 : 0;
    if (p->att_gmode && dp_tensor_core_mode() == 6 && att_bwd_tc_ok(dm)) {
        // tcgen05 / TMA digit-plane kernel (att_tc.cu): whole samples per CTA,
        // per-tile partials
        p->att_per_sample = 0;
        return launch_att_bwd_tc(dm, rows / dm.T, p->proj, p->proj_dig, p->proj_inv, p->encW, p->act_h, p->row_w,
                                 p->row_du, p->act_e, p->act_esc, tile_part, tile_partA, p->row_dhx, g.n_used, st);
    }
    if (p->att_gmode) {
        DP_CUDA_TRY(allow_big_smem((const void *)att_bwd_kernel<true, true>, smem));
        att_bwd_kernel<true, true><<<g.n_used, kThreads, smem, st>>>(
            dm, rows, g.per, p->proj, p->act_stat, p->act_h, p->encW, p->row_w, p->row_du, p->row_dq, p->partial,
            p->partA, tile_part, tile_partA, p->act_e, p->act_esc, 1, per_sample, params + p->dims.off.w_att,
            p->row_dhx, prep, params, p->act_p, p->act_choice, p->act_uc, p->row_du);
    } else if (p->act_e) {
        DP_CUDA_TRY(allow_big_smem((const void *)att_bwd_kernel<true>, smem));
        att_bwd_kernel<true><<<g.n_used, kThreads, smem, st>>>(dm, rows, g.per, p->enc_h, p->act_stat, p->row_q,
                                                               p->encW, p->row_w, p->row_du, p->row_dq, p->partial,
                                                               p->partA, tile_part, tile_partA, p->act_e, p->act_esc, 1,
                                                               per_sample, params + p->dims.off.w_att, p->row_dhx);
    } else {
        DP_CUDA_TRY(allow_big_smem((const void *)att_bwd_kernel<false>, smem));
        att_bwd_kernel<false><<<g.n_used, kThreads, smem, st>>>(dm, rows, g.per, p->enc_h, p->act_stat, p->row_q,
                                                                p->encW, p->row_w, p->row_du, p->row_dq, p->partial,
                                                                p->partA, tile_part, tile_partA, nullptr, nullptr, 1,
                                                                per_sample, params + p->dims.off.w_att, p->row_dhx);
    }
    DP_LAUNCH_CHECK();
    return DP_OK;
}

int run_att_fin(dp_policy *p, const double *params, double *grad, cudaStream_t st) {
    const PolicyDims &dm = p->dims;
    const int nb = ceil_div(dm.T * kH, 256);
    att_fin_kernel<<<nb + ceil_div(kH * dm.dd, 32), 256, 0, st>>>(dm, params, p->enc_h, p->a_tot, p->d_enc, grad, nb);
    DP_LAUNCH_CHECK();
    return DP_OK;
}

// B0 in the given mode (+ its reductions when it produces gradients)
int run_b0(dp_policy *p, const double *params, int rows, const double *adv, double *grad, int mode,
           cudaStream_t st) {
    const PolicyDims &dm = p->dims;
    const Grid g = persist_grid(rows, kTile);
    const size_t smem = sizeof(PrepSmem);
    DP_CUDA_TRY(allow_big_smem((const void *)row_prep_kernel, smem));
    row_prep_kernel<<<g.n_used, kThreads, smem, st>>>(dm, params, rows, g.per, adv, p->act_p, p->act_choice, p->act_u,
                                                      p->act_h, p->act_uc, p->row_q, p->row_w,
                                                      p->row_dhx, p->row_du, p->partial, mode,
                                                      !(mode == kRowsOnly && p->act_e && p->tile_part));
    DP_LAUNCH_CHECK();
    if (mode == kRowsOnly) return DP_OK;
    const int na = dm.D + dm.D * dm.dd + 2 * kH * dm.dd;
    double *part = p->partial;
    launch_reduce(part, g.n_used, na, dm.D, grad + dm.off.b_out, 0, st);
    DP_LAUNCH_CHECK();
    launch_reduce(part + dm.D, g.n_used, na, dm.D * dm.dd, grad + dm.off.dev_table, 0, st);
    DP_LAUNCH_CHECK();
    launch_reduce(part + dm.D + dm.D * dm.dd, g.n_used, na, kH * dm.dd, grad + dm.off.w_out, 0, st);
    DP_LAUNCH_CHECK();
    return DP_OK;
}

int run_b1f(dp_policy *p, const double *params, int rows, const double *adv, double *grad, int mode,
            cudaStream_t st) {
    const PolicyDims &dm = p->dims;
    const Grid g = tiles_grid(rows, kFinTile);
    const size_t smem = sizeof(FinSmem);
    DP_CUDA_TRY(allow_big_smem((const void *)row_fin_kernel, smem));
    row_fin_kernel<<<g.n_used, kThreads, smem, st>>>(dm, params, rows, g.per, p->act_h, p->row_dq, p->row_dhx,
                                                     p->partial, adv, mode);
    DP_LAUNCH_CHECK();
    if (mode == kRowsOnly) return DP_OK;
    launch_reduce(p->partial, g.n_used, kH * kH, kH * kH, grad + dm.off.w_att, 0, st);
    DP_LAUNCH_CHECK();
    return DP_OK;
}

// B2: decoder LSTM backward, per sample (inputs row_dhx; da in place of act_g)
int run_b2(dp_policy *p, const double *params, int K, cudaStream_t st) {
    const PolicyDims &dm = p->dims;
    int M = ceil_div(K, kNumSMs);
    if (M > kMaxSeqPerCta) M = kMaxSeqPerCta;
    const size_t smem = lstm_bwd_smem(M);
    const void *fn = lstm_bwd_fn(M);
    DP_CUDA_TRY(allow_big_smem(fn, smem));
    {
        int T = dm.T, n_seq = K;
        const double *Wh = params + dm.off.w_dec + (size_t)dm.dd * kG;
        const double *c_init = p->enc_c + (size_t)(dm.T - 1) * kH;
        const double *null = nullptr;
        const double *gin = p->act_g;
        int zero = 0;
        DP_CUDA_TRY(cudaMemsetAsync(p->da_colexp, 0, sizeof(int) * kG, st));
        void *args[] = {&T,       &n_seq,   &M,    &Wh,   &p->act_g, &p->act_c, &c_init, &p->row_dhx, &null,
                        &null,    &p->dh0,  &p->dc0, &gin, &null,     &null,     &null,   &zero, &p->da_colexp};
        DP_CUDA_TRY(cudaLaunchKernel(fn, dim3(ceil_div(K, M)), dim3(kLstmThreads), args, smem, st));
    }
    DP_LAUNCH_CHECK();
    return DP_OK;
}

// B3 on the main stream, B4 + B5 forked onto the side stream; adv == NULL: da/dh0/dc0 already scaled
// split_grads: also run the advantage-weighted B0 / B1f reductions on the main
// stream inside the fork window (they only need adv and the rows-pass outputs),
// concurrently with the sequential encoder backward.
int run_b345(dp_policy *p, const double *params, int K, const double *adv, double *grad, cudaStream_t st,
             bool split_grads = false) {
    const PolicyDims &dm = p->dims;
    const int T = dm.T, rows = K * T;
    double *part = p->partial;
    double *dx_scratch = part + (p->partial_elems - (size_t)T * dm.td - 4 * kH);
    double *dhc_sum = dx_scratch + (size_t)T * dm.td;
    // Fork: B4 + B5 (encoder backward: one CTA, sequential over T, then the
    // encoder weight gradients) run on the side stream while B3 fills the
    // other SMs.  Disjoint outputs (grad[w_enc,b_enc,type_table] vs
    // grad[w_dec,b_dec,dev_table]) and scratch (partial tail vs head).
    DP_CUDA_TRY(cudaEventRecord(p->ev_fork, st));
    DP_CUDA_TRY(cudaStreamWaitEvent(p->side, p->ev_fork, 0));
    {
        cudaStream_t ss = p->side;
        // encoder backward: reads the gate activations from enc_g, writes da to
        // da_enc, and sums the decoders' step-0 state gradients in its prologue
        const size_t smem = lstm_bwd_smem(1);
        if (g_lstm_clocks_on)
            lstm_bwd_kernel<1, true><<<1, kLstmThreads, smem, ss>>>(T, 1, 1, params + dm.off.w_enc + (size_t)dm.F * kG, p->da_enc,
                                                   p->enc_c, p->zeros, p->d_enc, nullptr, nullptr,
                                                   dhc_sum + 2 * kH, dhc_sum + 3 * kH, p->enc_g, p->dh0, p->dc0, adv,
                                                   K, nullptr);
        else
            lstm_bwd_kernel<1><<<1, kLstmThreads, smem, ss>>>(T, 1, 1, params + dm.off.w_enc + (size_t)dm.F * kG, p->da_enc,
                                                   p->enc_c, p->zeros, p->d_enc, nullptr, nullptr,
                                                   dhc_sum + 2 * kH, dhc_sum + 3 * kH, p->enc_g, p->dh0, p->dc0, adv,
                                                   K, nullptr);
        DP_LAUNCH_CHECK();
        // the encoder weight grads and the type-table chain both only need
        // da_enc: fork the former onto a second side stream
        DP_CUDA_TRY(cudaEventRecord(p->ev_fork2, ss));
        DP_CUDA_TRY(cudaStreamWaitEvent(p->side2, p->ev_fork2, 0));
        {
            const size_t xs = enc_wgrad_smem(T);
            DP_CUDA_TRY(allow_big_smem((const void *)enc_wgrad_kernel, xs));
            enc_wgrad_kernel<<<ceil_div(dm.F + kH + 1, kWgRows), kG, xs, p->side2>>>(dm, p->X, p->enc_h, p->da_enc,
                                                                                   grad);
        }
        DP_LAUNCH_CHECK();
        DP_CUDA_TRY(cudaEventRecord(p->ev_join2, p->side2));
        enc_dx_kernel<<<T, kG, 0, ss>>>(dm, params, p->da_enc, dx_scratch);
        DP_LAUNCH_CHECK();
        type_scatter_kernel<<<dm.V1, 256, 0, ss>>>(dm, p->occ_off, p->occ_t, p->type_off, dx_scratch, grad);
        DP_LAUNCH_CHECK();
        DP_CUDA_TRY(cudaStreamWaitEvent(ss, p->ev_join2, 0));
        DP_CUDA_TRY(cudaEventRecord(p->ev_join, ss));
    }
    if (split_grads) {
        // B0g + B1fg in one pass over the rows
        const Grid g = tiles_grid(rows, kTile);
        const int n_cta = ceil_div(ceil_div(rows, kTile), ceil_div(ceil_div(rows, kTile), kNumSMs));
        const int per = ceil_div(ceil_div(rows, kTile), n_cta);
        (void)g;
        const size_t smem = sizeof(AdvGradSmem);
        DP_CUDA_TRY(allow_big_smem((const void *)adv_grads_kernel, smem));
        const int nq = p->att_gmode ? 0 : kH;  // GM: W_att comes from G (gsum_fin_kernel)
        adv_grads_kernel<<<n_cta, kThreads, smem, st>>>(dm, rows, per, adv, p->act_h, p->row_dq, p->row_du, p->act_u,
                                                         p->act_p, p->act_choice, part, nq);
        DP_LAUNCH_CHECK();
        const size_t na = adv_grads_partial(dm);
        RedBuilder rb;
        rb.add(part, na, dm.D, grad + dm.off.b_out);
        rb.add(part + dm.D, na, dm.D * dm.dd, grad + dm.off.dev_table);
        rb.add(part + dm.D + dm.D * dm.dd, na, kH * dm.dd, grad + dm.off.w_out);
        if (nq) rb.add(part + dm.D + dm.D * dm.dd + kH * dm.dd, na, kH * kH, grad + dm.off.w_att);
        rb.launch(n_cta, 0, st);
        DP_LAUNCH_CHECK();
    }
    // B3: tcgen05 / TMA int8-digit GEMM (wgrad_tc.cu) where the shape allows,
    // else the DMMA kernel
    if (dp_tensor_core_mode() != 1 && dec_wgrad_tc_ok(dm)) {
        int n_chunks = 0;
        DP_TRY(launch_dec_wgrad_tc(dm, rows, p->act_h, p->enc_h, p->act_choice, p->act_g, p->da_colexp, adv, K, part,
                                   &n_chunks, st));
        const size_t stride = (size_t)(kH + dm.D + 1) * kG;
        RedBuilder rb;
        rb.add(part, stride, kH * kG, grad + dm.off.w_dec + (size_t)dm.dd * kG);
        rb.add(part + (size_t)kH * kG, stride, (dm.D + 1) * kG, p->gacc);
        rb.launch(n_chunks, 0, st);
        DP_LAUNCH_CHECK();
        dec_finalize_kernel<<<1 + ceil_div((dm.D + 1) * dm.dd, kG / 32), kG, 0, st>>>(dm, params, p->gacc, grad);
        DP_LAUNCH_CHECK();
    } else {
        const Grid g = tiles_grid(rows, kTile);
        const size_t smem = sizeof(double) * ((size_t)2 * kTile * (kWgHLd + kWgDLd) + (size_t)(dm.D + 1) * kG);
        DP_CUDA_TRY(allow_big_smem((const void *)dec_wgrad_kernel, smem));
        dec_wgrad_kernel<<<g.n_used, kThreads, smem, st>>>(dm, rows, g.per, p->act_h, p->enc_h, p->act_choice,
                                                           p->act_g, part, adv);
        DP_LAUNCH_CHECK();
        const size_t stride = (size_t)(kH + dm.D + 1) * kG;
        RedBuilder rb;
        rb.add(part, stride, kH * kG, grad + dm.off.w_dec + (size_t)dm.dd * kG);
        rb.add(part + (size_t)kH * kG, stride, (dm.D + 1) * kG, p->gacc);
        rb.launch(g.n_used, 0, st);
        DP_LAUNCH_CHECK();
        dec_finalize_kernel<<<1 + ceil_div((dm.D + 1) * dm.dd, kG / 32), kG, 0, st>>>(dm, params, p->gacc, grad);
        DP_LAUNCH_CHECK();
    }
    DP_CUDA_TRY(cudaStreamWaitEvent(st, p->ev_join, 0));
    return DP_OK;
}


}  // namespace

// Fused single pass (advantages known up front).
extern "C" int dp_policy_backward(dp_policy *p, const double *params, int32_t K, const double *adv, double *grad,
                                  void *stream) {
    DP_ENTRY();
    DP_REQUIRE(p && params && adv && grad, "dp_policy_backward: NULL argument");
    DP_REQUIRE(K >= 1 && K == p->last_K, "dp_policy_backward: K must equal the last decode's K");
    const PolicyDims &dm = p->dims;
    cudaStream_t st = (cudaStream_t)stream;
    const int T = dm.T, rows = K * T;
    DP_CUDA_TRY(cudaMemsetAsync(grad, 0, sizeof(double) * dm.off.total, st));
    p->rows_ready = 0;
    DP_TRY(run_b0(p, params, rows, adv, grad, kFused, st));
    {
        const Grid g = att_grid(K, T, false);
        const size_t smem = sizeof(AttSmem);
        DP_TRY(launch_att(p, params, g, smem, rows, nullptr, nullptr, st));
        launch_reduce(p->partial, g.n_used, (size_t)T * kH, T * kH, p->d_enc, 0, st);
        DP_LAUNCH_CHECK();
        launch_reduce(p->partA, g.n_used, (size_t)T * dm.dd, T * dm.dd, p->a_tot, 0, st);
        DP_LAUNCH_CHECK();
        DP_TRY(run_att_fin(p, params, grad, st));
    }
    DP_TRY(run_b1f(p, params, rows, nullptr, grad, kFusedGrads, st));
    DP_TRY(run_b2(p, params, K, st));
    return run_b345(p, params, K, nullptr, grad, st);
}

// Advantage-independent half: everything per sample that is linear in adv,
// computed with adv := 1 (B0, attention backward with alpha/ds stored, B1f,
// the decoder LSTM backward).  Enqueue it concurrently with scoring.
extern "C" int dp_policy_backward_rows(dp_policy *p, const double *params, int32_t K, void *stream) {
    DP_ENTRY();
    DP_REQUIRE(p && params, "dp_policy_backward_rows: NULL argument");
    DP_REQUIRE(K >= 1 && K == p->last_K, "dp_policy_backward_rows: K must equal the last decode's K");
    p->rows_ready = 0;
    if (!p->tile_part) return DP_OK;  // partials too large: grads() runs the fused pass
    const PolicyDims &dm = p->dims;
    cudaStream_t st = (cudaStream_t)stream;
    const int rows = K * dm.T;
    // GM: the attention backward forms row_prep's per-row outputs per tile itself
    const bool merged = att_prep_merged(p);
    if (!merged) DP_TRY(run_b0(p, params, rows, nullptr, nullptr, kRowsOnly, st));
    {
        const Grid g = att_grid(K, dm.T, true);
        const size_t smem = sizeof(AttSmem);
        DP_TRY(launch_att(p, params, g, smem, rows, p->tile_part, p->tile_partA, st, merged ? 1 : 0));
    }
    DP_CUDA_TRY(cudaEventRecord(p->ev_att, st));  // the grads pass's reductions may start here
    DP_TRY(run_b2(p, params, K, st));
    DP_CUDA_TRY(cudaEventRecord(p->ev_rows, st));
    p->rows_ready = K;
    return DP_OK;
}

// Advantage-weighted half: cross-sample sums of the per-row quantities left
// by dp_policy_backward_rows (falls back to the fused pass if that did not run).
extern "C" int dp_policy_backward_grads(dp_policy *p, const double *params, int32_t K, const double *adv,
                                        double *grad, void *stream) {
    DP_ENTRY();
    DP_REQUIRE(p && params && adv && grad, "dp_policy_backward_grads: NULL argument");
    if (p->rows_ready != K) return dp_policy_backward(p, params, K, adv, grad, stream);
    const PolicyDims &dm = p->dims;
    cudaStream_t st = (cudaStream_t)stream;
    const int T = dm.T, rows = K * T;
    // the advantage-weighted attention sums need only the attention backward:
    // they run beside the decoder LSTM backward; the rest waits for the rows pass
    DP_CUDA_TRY(cudaStreamWaitEvent(st, p->ev_att, 0));
    DP_CUDA_TRY(cudaMemsetAsync(grad, 0, sizeof(double) * dm.off.total, st));
    {
        // per-sample partials (1 unit per sample) or per-tile (tps units per sample)
        const int tps = p->att_per_sample ? 1 : (T + kAttTile - 1) / kAttTile;
        RedBuilder rb;
        rb.add(p->tile_part, (size_t)T * kH, T * kH, p->att_gmode ? p->gsum : p->d_enc);
        rb.add(p->tile_partA, (size_t)T * dm.dd, T * dm.dd, p->a_tot);
        rb.launch(K * tps, 0, st, adv, tps);
        DP_LAUNCH_CHECK();
        if (p->att_gmode) {
            const int nb = ceil_div(T, kGfRows);
            gsum_fin_kernel<<<nb + kH + ceil_div(kH * dm.dd, kH), 256, 0, st>>>(dm, params, nb, p->gsum, p->a_tot,
                                                                              p->enc_h, p->d_enc, grad);
            DP_LAUNCH_CHECK();
        }
    }
    if (!p->att_gmode) DP_TRY(run_att_fin(p, params, grad, st));
    DP_CUDA_TRY(cudaStreamWaitEvent(st, p->ev_rows, 0));
    // the encoder backward (sequential) forks first; B0 / B1f grads and B3 fill the other SMs
    return run_b345(p, params, K, adv, grad, st, true);
}

// Debug: 1 = run the DMMA / SIMT kernels where a tcgen05 path exists (A/B parity runs);
// 2 = tcgen05 with a TMEM drain every 3 steps (exercises the multi-segment epilogue);
// 3 / 4 / 5 = timing ablations of the tcgen05 weight gradient (no conversion / no TMA / neither; wrong results);
// 6 = also the attention backward on tcgen05 (att_tc.cu; measured slower than the DMMA kernel at C3).
extern "C" int dp_debug_tensor_core(int32_t mode) {
    DP_ENTRY();
    DP_REQUIRE(mode >= 0 && mode <= 6, "dp_debug_tensor_core: mode must be 0..6");
    dp::g_tc_mode = mode;
    return DP_OK;
}
