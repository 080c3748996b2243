// Policy-gradient backward on sm_100a: grad = sum_k adv[k] * d log p_k / d theta.
//
// Reference: grad_log_prob (/root/reference/pkg/src/devplace/policy.py:351-409,
// _lstm_backward 236-253) called per sample by reinforce_update
// (pkg/trainer.py:138-154), which forms sum_k (r_k - b) * g_k.
//
// Restructuring — every step is linear in the per-sample
// advantage, so adv[k] scales dz at the top and all cross-sample sums happen
// inside the kernels:
//   B0 row_prep    (parallel over rows (k,t)): dz, du, dhc -> dh_out, dctx;
//                  q = W_att^T h; w = ctx.dctx (== alpha.dalpha); grads of
//                  b_out, dev_table[:D] (dz x u), w_out (hc x du)
//   B1 att_bwd     (parallel, tiled fp64 GEMMs over rows x T-chunks):
//                  recompute s, alpha (forward softmax stats), dalpha = enc.dctx,
//                  ds = alpha*(dalpha - w); dq += ds@enc;
//                  d_enc += alpha^T dctx + ds^T q  (== d_enc + d_proj@W_att of
//                  the reference, with proj@h restated as enc@(W_att^T h))
//   B1f row_fin    (parallel): dh_ext = dh_out + W_att dq; w_att grad += h x dq
//   B2 dec_lstm    (sequential over t, parallel over samples): LSTM backward,
//                  dh_prev = W_dec[dd:] da; stores da per row
//   B3 dec_wgrad   (parallel split-K): w_dec[dd:] += h_prev x da; per input row
//                  sums of da give b_dec, w_dec[:dd] and dev_table row grads
//   B4 enc_lstm    (sequential, ONE sequence): the encoder is shared by all
//                  samples, so its backward runs once on the summed inputs
//                  (the reference runs it per sample)
//   B5 enc_wgrad   w_enc, b_enc, type_table (np.add.at order)
// Deterministic: fixed partition + ordered reductions, no float atomics.

#include <math.h>

#include "policy.cuh"

namespace dp {

namespace {

constexpr int kRowsPerWarpBatch = 8;   // B0/B1f: one row per warp per batch
constexpr int kTile = 32;              // B1: rows per tile
constexpr int kChunk = 64;             // B1: enc rows per chunk
constexpr int kPad = 65;

__device__ __forceinline__ double warp_sum(double v) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// ------------------------------------------------------------------ B0
// grad partial layout per CTA: [b_out (D) | dev_table[:D] (D*dd) | w_out (128*dd)]
__global__ void __launch_bounds__(kThreads) row_prep_kernel(
    PolicyDims dm, const double *__restrict__ P, int rows, int rows_per_cta, const double *__restrict__ adv,
    const double *__restrict__ act_p, const uint8_t *__restrict__ choice, const double *__restrict__ act_u,
    const double *__restrict__ act_h, const double *__restrict__ act_ctx, double *__restrict__ row_q,
    double *__restrict__ row_dctx, double *__restrict__ row_w, double *__restrict__ row_dhx,
    double *__restrict__ partial) {
    extern __shared__ __align__(16) double sm0[];
    __shared__ double s_dz[kRowsPerWarpBatch][kMaxD];
    __shared__ double s_u[kRowsPerWarpBatch][kMaxDD];
    __shared__ double s_du[kRowsPerWarpBatch][kMaxDD];
    __shared__ double s_hc[kRowsPerWarpBatch][2 * kH];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int D = dm.D, dd = dm.dd, T = dm.T;
    double *watt = sm0;                  // [64*64]
    double *wout = watt + kH * kH;       // [128*dd]
    double *devt = wout + 2 * kH * dd;   // [D*dd]
    for (int i = tid; i < kH * kH; i += kThreads) watt[i] = P[dm.off.w_att + i];
    for (int i = tid; i < 2 * kH * dd; i += kThreads) wout[i] = P[dm.off.w_out + i];
    for (int i = tid; i < D * dd; i += kThreads) devt[i] = P[dm.off.dev_table + i];
    const int n_acc = D + D * dd + 2 * kH * dd;
    // thread-owned accumulators (strided ownership of the partial layout)
    constexpr int kMaxOwn = (kMaxD + kMaxD * kMaxDD + 2 * kH * kMaxDD + kThreads - 1) / kThreads;
    double acc[kMaxOwn];
#pragma unroll
    for (int i = 0; i < kMaxOwn; i++) acc[i] = 0.0;
    const int r0 = blockIdx.x * rows_per_cta, r1 = min(rows, r0 + rows_per_cta);
    __syncthreads();
    for (int rb = r0; rb < r1; rb += kRowsPerWarpBatch) {
        const int row = rb + warp;
        const bool live = row < r1;
        if (live) {
            const int k = row / T;
            const double a = adv[k];
            const int c = choice[row];
            double dz = 0.0;
            if (lane < D) {
                dz = -act_p[(size_t)row * D + lane];
                if (lane == c) dz += 1.0;
                dz = a * dz;
                s_dz[warp][lane] = dz;
            }
            if (lane < dd) s_u[warp][lane] = act_u[(size_t)row * dd + lane];
            const double *h = act_h + (size_t)row * kH;
            const double *cx = act_ctx + (size_t)row * kH;
            s_hc[warp][lane] = h[lane];
            s_hc[warp][lane + 32] = h[lane + 32];
            s_hc[warp][lane + 64] = cx[lane];
            s_hc[warp][lane + 96] = cx[lane + 32];
            __syncwarp();
            // du = dev_table[:D]^T dz
            double du = 0.0;
            if (lane < dd) {
                for (int dv = 0; dv < D; dv++) du = fma(devt[dv * dd + lane], s_dz[warp][dv], du);
                s_du[warp][lane] = du;
            }
            __syncwarp();
            // dhc = w_out @ du  -> dh_out (rows 0..63), dctx (rows 64..127)
            double dhc[4];
#pragma unroll
            for (int r = 0; r < 4; r++) {
                const int i = lane + 32 * r;
                double v = 0.0;
                for (int o = 0; o < dd; o++) v = fma(wout[i * dd + o], s_du[warp][o], v);
                dhc[r] = v;
            }
            row_dhx[(size_t)row * kH + lane] = dhc[0];
            row_dhx[(size_t)row * kH + lane + 32] = dhc[1];
            row_dctx[(size_t)row * kH + lane] = dhc[2];
            row_dctx[(size_t)row * kH + lane + 32] = dhc[3];
            // w = ctx . dctx  (== alpha . dalpha)
            const double wv = warp_sum(fma(s_hc[warp][64 + lane], dhc[2], s_hc[warp][96 + lane] * dhc[3]));
            if (lane == 0) row_w[row] = wv;
            // q = W_att^T h
#pragma unroll
            for (int r = 0; r < 2; r++) {
                const int j = lane + 32 * r;
                double q0 = 0.0, q1 = 0.0;
                for (int l = 0; l < kH; l += 2) {
                    q0 = fma(watt[l * kH + j], s_hc[warp][l], q0);
                    q1 = fma(watt[(l + 1) * kH + j], s_hc[warp][l + 1], q1);
                }
                row_q[(size_t)row * kH + j] = q0 + q1;
            }
        } else {
            if (lane < D) s_dz[warp][lane] = 0.0;
            if (lane < dd) {
                s_u[warp][lane] = 0.0;
                s_du[warp][lane] = 0.0;
            }
            for (int i = lane; i < 2 * kH; i += 32) s_hc[warp][i] = 0.0;
        }
        __syncthreads();
        // accumulate owned grad elements over the batch's rows (in row order)
#pragma unroll
        for (int s = 0; s < kMaxOwn; s++) {
            const int e = tid + s * kThreads;
            if (e < n_acc) {
                double v = acc[s];
                for (int w8 = 0; w8 < kRowsPerWarpBatch; w8++) {
                    if (e < D) {
                        v += s_dz[w8][e];
                    } else if (e < D + D * dd) {
                        const int dv = (e - D) / dd, o = (e - D) % dd;
                        v = fma(s_dz[w8][dv], s_u[w8][o], v);
                    } else {
                        const int i = (e - D - D * dd) / dd, o = (e - D - D * dd) % dd;
                        v = fma(s_hc[w8][i], s_du[w8][o], v);
                    }
                }
                acc[s] = v;
            }
        }
        __syncthreads();
    }
#pragma unroll
    for (int s = 0; s < kMaxOwn; s++) {
        const int e = tid + s * kThreads;
        if (e < n_acc) partial[(size_t)blockIdx.x * n_acc + e] = acc[s];
    }
}

// ------------------------------------------------------------------ B1
struct AttSmem {
    double enc[kChunk * kPad];
    double q[kTile * kPad];
    double dc[kTile * kPad];
    double al[kTile * kPad];
    double ds[kTile * kPad];
    double mx[kTile], sm[kTile], w[kTile];
};

__global__ void __launch_bounds__(kThreads) att_bwd_kernel(
    PolicyDims dm, int rows, int tiles_per_cta, const double *__restrict__ enc_h,
    const double *__restrict__ act_stat, const double *__restrict__ row_q, const double *__restrict__ row_dctx,
    const double *__restrict__ row_w, double *__restrict__ row_dq, double *__restrict__ partial) {
    extern __shared__ __align__(16) double smraw[];
    AttSmem &S = *reinterpret_cast<AttSmem *>(smraw);
    const int tid = threadIdx.x;
    const int T = dm.T;
    const int n_chunks = (T + kChunk - 1) / kChunk;
    const int tile0 = blockIdx.x * tiles_per_cta;
    const int n_tiles_total = (rows + kTile - 1) / kTile;
    const int tile1 = min(n_tiles_total, tile0 + tiles_per_cta);
    // S/DA micro-tile: row = tid>>3, i in {ib + 8*ii}
    const int sr = tid >> 3, ib = tid & 7;
    // dE micro-tile: i in {ei + 16*a}, j in {ej + 16*b} (a,b < 4)
    const int ei = tid >> 4, ej = tid & 15;
    for (int ch = 0; ch < n_chunks; ch++) {
        const int i0 = ch * kChunk;
        for (int x = tid; x < kChunk * kH; x += kThreads) {
            const int i = x >> 6, j = x & 63;
            S.enc[i * kPad + j] = (i0 + i < T) ? enc_h[(size_t)(i0 + i) * kH + j] : 0.0;
        }
        double dE[4][4];
#pragma unroll
        for (int a = 0; a < 4; a++)
#pragma unroll
            for (int b = 0; b < 4; b++) dE[a][b] = 0.0;
        for (int tl = tile0; tl < tile1; tl++) {
            const int rb = tl * kTile;
            __syncthreads();
            for (int x = tid; x < kTile * kH; x += kThreads) {
                const int r = x >> 6, j = x & 63;
                const int row = rb + r;
                const bool ok = row < rows;
                S.q[r * kPad + j] = ok ? row_q[(size_t)row * kH + j] : 0.0;
                S.dc[r * kPad + j] = ok ? row_dctx[(size_t)row * kH + j] : 0.0;
            }
            if (tid < kTile) {
                const int row = rb + tid;
                const bool ok = row < rows;
                S.mx[tid] = ok ? act_stat[(size_t)row * 2] : 0.0;
                S.sm[tid] = ok ? act_stat[(size_t)row * 2 + 1] : 1.0;
                S.w[tid] = ok ? row_w[row] : 0.0;
            }
            __syncthreads();
            // S = Q enc^T, DA = DCTX enc^T over this chunk
            {
                double sv[8], dv[8];
#pragma unroll
                for (int ii = 0; ii < 8; ii++) sv[ii] = dv[ii] = 0.0;
                const double *qr = S.q + sr * kPad;
                const double *dr = S.dc + sr * kPad;
#pragma unroll 4
                for (int j = 0; j < kH; j++) {
                    const double qj = qr[j], dj = dr[j];
#pragma unroll
                    for (int ii = 0; ii < 8; ii++) {
                        const double e = S.enc[(ib + 8 * ii) * kPad + j];
                        sv[ii] = fma(qj, e, sv[ii]);
                        dv[ii] = fma(dj, e, dv[ii]);
                    }
                }
                const double m = S.mx[sr], l = S.sm[sr], w = S.w[sr];
#pragma unroll
                for (int ii = 0; ii < 8; ii++) {
                    const int i = ib + 8 * ii;
                    double al = 0.0, ds = 0.0;
                    if (i0 + i < T) {
                        al = exp(sv[ii] - m) / l;
                        ds = al * (dv[ii] - w);
                    }
                    S.al[sr * kPad + i] = al;
                    S.ds[sr * kPad + i] = ds;
                }
            }
            __syncthreads();
            // dq[row, j] += sum_i ds[row, i] enc[i, j]
            {
                const int row = rb + sr;
                double acc[8];
#pragma unroll
                for (int jj = 0; jj < 8; jj++) acc[jj] = 0.0;
                const double *dsr = S.ds + sr * kPad;
#pragma unroll 4
                for (int i = 0; i < kChunk; i++) {
                    const double d = dsr[i];
#pragma unroll
                    for (int jj = 0; jj < 8; jj++) acc[jj] = fma(d, S.enc[i * kPad + ib + 8 * jj], acc[jj]);
                }
                if (row < rows) {
#pragma unroll
                    for (int jj = 0; jj < 8; jj++) {
                        double *dst = row_dq + (size_t)row * kH + ib + 8 * jj;
                        *dst = ch == 0 ? acc[jj] : *dst + acc[jj];
                    }
                }
            }
            // dE[i, j] += sum_r al[r, i] dc[r, j] + ds[r, i] q[r, j]
#pragma unroll 2
            for (int r = 0; r < kTile; r++) {
                double av[4], sv4[4], dcv[4], qv[4];
#pragma unroll
                for (int a = 0; a < 4; a++) {
                    av[a] = S.al[r * kPad + ei + 16 * a];
                    sv4[a] = S.ds[r * kPad + ei + 16 * a];
                }
#pragma unroll
                for (int b = 0; b < 4; b++) {
                    dcv[b] = S.dc[r * kPad + ej + 16 * b];
                    qv[b] = S.q[r * kPad + ej + 16 * b];
                }
#pragma unroll
                for (int a = 0; a < 4; a++)
#pragma unroll
                    for (int b = 0; b < 4; b++) dE[a][b] = fma(sv4[a], qv[b], fma(av[a], dcv[b], dE[a][b]));
            }
        }
        // write this CTA's partial for the chunk
#pragma unroll
        for (int a = 0; a < 4; a++) {
            const int i = i0 + ei + 16 * a;
            if (i < T) {
#pragma unroll
                for (int b = 0; b < 4; b++)
                    partial[((size_t)blockIdx.x * T + i) * kH + ej + 16 * b] = dE[a][b];
            }
        }
        __syncthreads();
    }
}

// ------------------------------------------------------------------ B1f
// dh_ext = dh_out + W_att dq ; partial w_att grad (64x64) += h x dq
__global__ void __launch_bounds__(kThreads) row_fin_kernel(PolicyDims dm, const double *__restrict__ P, int rows,
                                                           int rows_per_cta, const double *__restrict__ act_h,
                                                           const double *__restrict__ row_dq,
                                                           double *__restrict__ row_dhx, double *__restrict__ partial) {
    __shared__ double watt[kH * kH];
    __shared__ double s_h[kRowsPerWarpBatch][kH];
    __shared__ double s_q[kRowsPerWarpBatch][kH];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int i = tid; i < kH * kH; i += kThreads) watt[i] = P[dm.off.w_att + i];
    double acc[16];
#pragma unroll
    for (int s = 0; s < 16; s++) acc[s] = 0.0;
    const int r0 = blockIdx.x * rows_per_cta, r1 = min(rows, r0 + rows_per_cta);
    __syncthreads();
    for (int rb = r0; rb < r1; rb += kRowsPerWarpBatch) {
        const int row = rb + warp;
        if (row < r1) {
            const double *dq = row_dq + (size_t)row * kH;
            const double *h = act_h + (size_t)row * kH;
            s_q[warp][lane] = dq[lane];
            s_q[warp][lane + 32] = dq[lane + 32];
            s_h[warp][lane] = h[lane];
            s_h[warp][lane + 32] = h[lane + 32];
            __syncwarp();
#pragma unroll
            for (int r = 0; r < 2; r++) {
                const int l = lane + 32 * r;
                double v0 = 0.0, v1 = 0.0;
                for (int j = 0; j < kH; j += 2) {
                    v0 = fma(watt[l * kH + j], s_q[warp][j], v0);
                    v1 = fma(watt[l * kH + j + 1], s_q[warp][j + 1], v1);
                }
                row_dhx[(size_t)row * kH + l] += v0 + v1;
            }
        } else {
            s_q[warp][lane] = s_q[warp][lane + 32] = 0.0;
            s_h[warp][lane] = s_h[warp][lane + 32] = 0.0;
        }
        __syncthreads();
#pragma unroll
        for (int s = 0; s < 16; s++) {
            const int e = tid + s * kThreads;  // w_att grad element (l, j)
            const int l = e >> 6, j = e & 63;
            double v = acc[s];
            for (int w8 = 0; w8 < kRowsPerWarpBatch; w8++) v = fma(s_h[w8][l], s_q[w8][j], v);
            acc[s] = v;
        }
        __syncthreads();
    }
#pragma unroll
    for (int s = 0; s < 16; s++) partial[(size_t)blockIdx.x * kH * kH + tid + s * kThreads] = acc[s];
}

// ------------------------------------------------------------------ B2 / B4
// Sequential LSTM backward (pkg/policy.py:236-253) for M sequences per CTA.
// thread (r = tid>>2, part = tid&3) keeps W_h[r, part*64 : part*64+64] in
// registers; dh_prev[r] = sum over 4 parts (shuffle).  In-place: the gate
// activations of each row are replaced by da.
__global__ void __launch_bounds__(kThreads, 1) lstm_bwd_kernel(
    int T, int n_seq, int M, const double *__restrict__ Wh /* [64 x 256] row-major, ld 256 */,
    double *__restrict__ gates /* [seq][T][256] in: i,f,o,g  out: da */, const double *__restrict__ cst /* [seq][T][64] */,
    const double *__restrict__ c_init /* [64] c before step 0 */, const double *__restrict__ dh_ext /* [seq][T][64] */,
    const double *__restrict__ dh_in /* [seq][64] or NULL */, const double *__restrict__ dc_in,
    double *__restrict__ dh_out /* [seq][64] */, double *__restrict__ dc_out) {
    extern __shared__ __align__(16) double sm[];
    double *s_dh = sm;                   // [M][64]
    double *s_dc = s_dh + M * kH;        // [M][64]
    double *s_da = s_dc + M * kH;        // [M][256]
    const int tid = threadIdx.x, lane = tid & 31;
    const int q0 = blockIdx.x * M;
    const int Mb = min(M, n_seq - q0);
    const int r = tid >> 2, part = tid & 3;
    double w[kH];
#pragma unroll
    for (int i = 0; i < kH; i++) w[i] = Wh[(size_t)r * kG + part * kH + i];
    for (int x = tid; x < Mb * kH; x += kThreads) {
        const int m = x >> 6, u = x & 63;
        s_dh[x] = dh_in ? dh_in[(size_t)(q0 + m) * kH + u] : 0.0;
        s_dc[x] = dc_in ? dc_in[(size_t)(q0 + m) * kH + u] : 0.0;
    }
    __syncthreads();
    for (int t = T - 1; t >= 0; t--) {
        for (int x = tid; x < Mb * kH; x += kThreads) {
            const int m = x >> 6, u = x & 63;
            const size_t row = (size_t)(q0 + m) * T + t;
            double *g = gates + row * kG;
            const double iv = g[u], fv = g[kH + u], ov = g[2 * kH + u], gv = g[3 * kH + u];
            const double c = cst[row * kH + u];
            const double cp = t > 0 ? cst[(row - 1) * kH + u] : c_init[u];
            const double dh = s_dh[x] + dh_ext[row * kH + u];
            const double tc = tanh(c);
            const double d_o = dh * tc;
            const double dcv = s_dc[x] + dh * ov * (1.0 - tc * tc);
            const double di = dcv * gv;
            const double dg = dcv * iv;
            const double df = dcv * cp;
            s_dc[x] = dcv * fv;
            const double da_i = di * iv * (1.0 - iv);
            const double da_f = df * fv * (1.0 - fv);
            const double da_o = d_o * ov * (1.0 - ov);
            const double da_g = dg * (1.0 - gv * gv);
            double *sd = s_da + m * kG;
            sd[u] = da_i;
            sd[kH + u] = da_f;
            sd[2 * kH + u] = da_o;
            sd[3 * kH + u] = da_g;
            g[u] = da_i;
            g[kH + u] = da_f;
            g[2 * kH + u] = da_o;
            g[3 * kH + u] = da_g;
        }
        __syncthreads();
        for (int m = 0; m < Mb; m++) {
            const double *sd = s_da + m * kG + part * kH;
            double a0 = 0.0, a1 = 0.0;
#pragma unroll
            for (int i = 0; i < kH; i += 2) {
                a0 = fma(w[i], sd[i], a0);
                a1 = fma(w[i + 1], sd[i + 1], a1);
            }
            double v = a0 + a1;
            v += __shfl_xor_sync(0xffffffffu, v, 1);
            v += __shfl_xor_sync(0xffffffffu, v, 2);
            if (part == 0) s_dh[m * kH + r] = v;
        }
        __syncthreads();
    }
    (void)lane;
    for (int x = tid; x < Mb * kH; x += kThreads) {
        const int m = x >> 6, u = x & 63;
        dh_out[(size_t)(q0 + m) * kH + u] = s_dh[x];
        dc_out[(size_t)(q0 + m) * kH + u] = s_dc[x];
    }
}

// ------------------------------------------------------------------ B3
// partial per CTA: [Hg (64 x 256) | DAsum ((D+1) x 256)]
__global__ void __launch_bounds__(kThreads) dec_wgrad_kernel(PolicyDims dm, int rows, int rows_per_cta,
                                                             const double *__restrict__ act_h,
                                                             const double *__restrict__ enc_h,
                                                             const uint8_t *__restrict__ choice,
                                                             const double *__restrict__ da,
                                                             double *__restrict__ partial) {
    __shared__ double s_h[kTile][kH];
    __shared__ int s_prev[kTile];
    extern __shared__ __align__(16) double s_dasum[];  // [(D+1)][256] thread-owned columns
    const int tid = threadIdx.x;
    const int T = dm.T, D = dm.D;
    double acc[kH];
#pragma unroll
    for (int l = 0; l < kH; l++) acc[l] = 0.0;
    for (int p = 0; p <= D; p++) s_dasum[p * kG + tid] = 0.0;
    const int r0 = blockIdx.x * rows_per_cta, r1 = min(rows, r0 + rows_per_cta);
    for (int rb = r0; rb < r1; rb += kTile) {
        __syncthreads();
        for (int x = tid; x < kTile * kH; x += kThreads) {
            const int r = x >> 6, l = x & 63;
            const int row = rb + r;
            double v = 0.0;
            if (row < r1) {
                const int t = row % T;
                v = t > 0 ? act_h[(size_t)(row - 1) * kH + l] : enc_h[(size_t)(T - 1) * kH + l];
            }
            s_h[r][l] = v;
        }
        if (tid < kTile) {
            const int row = rb + tid;
            int pv = D;
            if (row < r1 && row % T > 0) pv = choice[row - 1];
            s_prev[tid] = pv;
        }
        __syncthreads();
        const int nr = min(kTile, r1 - rb);
        for (int r = 0; r < nr; r++) {
            const double d = da[(size_t)(rb + r) * kG + tid];
#pragma unroll
            for (int l = 0; l < kH; l++) acc[l] = fma(s_h[r][l], d, acc[l]);
            s_dasum[s_prev[r] * kG + tid] += d;
        }
    }
    const size_t base = (size_t)blockIdx.x * (kH + D + 1) * kG;
#pragma unroll
    for (int l = 0; l < kH; l++) partial[base + (size_t)l * kG + tid] = acc[l];
    for (int p = 0; p <= D; p++) partial[base + (size_t)(kH + p) * kG + tid] = s_dasum[p * kG + tid];
}

// ------------------------------------------------------------------ reductions
// dst[e] (+)= sum_c src[c * stride + e] (c ascending)
__global__ void reduce_partials_kernel(const double *__restrict__ src, int n_cta, size_t stride, int n,
                                       double *__restrict__ dst, int accumulate) {
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= n) return;
    double v = src[e];
    for (int c = 1; c < n_cta; c++) v += src[(size_t)c * stride + e];
    dst[e] = accumulate ? dst[e] + v : v;
}

// B3 finalize: b_dec = sum_p DAsum[p]; w_dec[:dd] = sum_p dev_table[p] x DAsum[p];
// dev_table[p] += W_dec[:dd] . DAsum[p]
__global__ void dec_finalize_kernel(PolicyDims dm, const double *__restrict__ P, const double *__restrict__ dasum,
                                    double *__restrict__ grad) {
    const int tid = threadIdx.x;  // 256 threads: gate column
    const int D = dm.D, dd = dm.dd;
    double b = 0.0;
    for (int p = 0; p <= D; p++) b += dasum[p * kG + tid];
    grad[dm.off.b_dec + tid] = b;
    for (int i = 0; i < dd; i++) {
        double v = 0.0;
        for (int p = 0; p <= D; p++) v = fma(P[dm.off.dev_table + p * dd + i], dasum[p * kG + tid], v);
        grad[dm.off.w_dec + (size_t)i * kG + tid] = v;
    }
    // dev_table rows: one (p, i) per thread
    for (int x = tid; x < (D + 1) * dd; x += blockDim.x) {
        const int p = x / dd, i = x % dd;
        double v = 0.0;
        for (int j = 0; j < kG; j++) v = fma(P[dm.off.w_dec + (size_t)i * kG + j], dasum[p * kG + j], v);
        grad[dm.off.dev_table + x] += v;
    }
}

// sum over samples of the decoder's dh/dc at step 0 -> encoder final state grads
__global__ void sum_rows_kernel(const double *__restrict__ src, int n_rows, double *__restrict__ dst) {
    const int j = threadIdx.x;  // 64
    double v = src[j];
    for (int r = 1; r < n_rows; r++) v += src[(size_t)r * kH + j];
    dst[j] = v;
}

// B5: w_enc / b_enc grads (contraction over T) and the type-embedding scatter.
__global__ void enc_wgrad_kernel(PolicyDims dm, const double *__restrict__ X, const double *__restrict__ enc_h,
                                 const double *__restrict__ da_enc, double *__restrict__ grad) {
    const int j = threadIdx.x;   // gate column
    const int r = blockIdx.x;    // row of w_enc (0..F+H-1), or F+H for b_enc
    const int T = dm.T, F = dm.F;
    double v = 0.0;
    if (r == F + kH) {
        for (int t = 0; t < T; t++) v += da_enc[(size_t)t * kG + j];
        grad[dm.off.b_enc + j] = v;
        return;
    }
    for (int t = 0; t < T; t++) {
        double x;
        if (r < F) x = X[(size_t)t * F + r];
        else x = t > 0 ? enc_h[(size_t)(t - 1) * kH + (r - F)] : 0.0;
        v = fma(x, da_enc[(size_t)t * kG + j], v);
    }
    grad[dm.off.w_enc + (size_t)r * kG + j] = v;
}

// dx_t[f] = W_enc[f, :] . da_enc[t]   (f < type_dim)
__global__ void enc_dx_kernel(PolicyDims dm, const double *__restrict__ P, const double *__restrict__ da_enc,
                              double *__restrict__ dx) {
    const int idx = blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= dm.T * dm.td) return;
    const int t = idx / dm.td, f = idx % dm.td;
    double v = 0.0;
    for (int j = 0; j < kG; j++) v = fma(P[dm.off.w_enc + (size_t)f * kG + j], da_enc[(size_t)t * kG + j], v);
    dx[idx] = v;
}

// np.add.at(type_table, idx_t, dx_t / len(idx_t)) in (t, position) order
// (pkg/policy.py:405-407): thread (v, f) walks its occurrence list.
__global__ void type_scatter_kernel(PolicyDims dm, const int32_t *__restrict__ occ_off,
                                    const int32_t *__restrict__ occ_t, const int32_t *__restrict__ type_off,
                                    const double *__restrict__ dx, double *__restrict__ grad) {
    const int idx = blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= dm.V1 * dm.td) return;
    const int v = idx / dm.td, f = idx % dm.td;
    double s = 0.0;
    for (int o = occ_off[v]; o < occ_off[v + 1]; o++) {
        const int t = occ_t[o];
        const double len = (double)(type_off[t + 1] - type_off[t]);
        s = s + dx[(size_t)t * dm.td + f] / len;
    }
    grad[dm.off.type_table + idx] = s;
}

int n_cta_for(int rows, int min_rows) {
    int n = ceil_div(rows, min_rows);
    if (n > 2 * kNumSMs) n = 2 * kNumSMs;
    return n < 1 ? 1 : n;
}

}  // namespace
}  // namespace dp

using namespace dp;

size_t dp_backward_partial_elems(const dp_policy *p) {
    const PolicyDims &dm = p->dims;
    const size_t ncta = 2 * kNumSMs;
    size_t a = ncta * (size_t)(dm.D + dm.D * dm.dd + 2 * kH * dm.dd);
    size_t b = ncta * (size_t)dm.T * kH;
    size_t c = ncta * (size_t)kH * kH;
    size_t d = ncta * (size_t)(kH + dm.D + 1) * kG;
    size_t m = a > b ? a : b;
    m = m > c ? m : c;
    m = m > d ? m : d;
    return m + (size_t)dm.T * dm.td + 2 * kH;  // + dx scratch + (dh, dc) sums
}

extern "C" int dp_policy_backward(dp_policy *p, const double *params, int32_t K, const double *adv, double *grad,
                                  void *stream) {
    DP_ENTRY();
    DP_REQUIRE(p && params && adv && grad, "dp_policy_backward: NULL argument");
    DP_REQUIRE(K >= 1 && K == p->last_K, "dp_policy_backward: K must equal the last decode's K");
    const PolicyDims &dm = p->dims;
    cudaStream_t st = (cudaStream_t)stream;
    const int T = dm.T;
    const int rows = K * T;
    double *part = p->partial;
    double *dx_scratch = part + (p->partial_elems - (size_t)T * dm.td - 2 * kH);
    double *dhc_sum = dx_scratch + (size_t)T * dm.td;
    DP_CUDA_TRY(cudaMemsetAsync(grad, 0, sizeof(double) * dm.off.total, st));

    // B0
    {
        const int n = n_cta_for(rows, 64);
        const int rpc = ceil_div(rows, n);
        const size_t smem = sizeof(double) * (kH * kH + 2 * kH * dm.dd + dm.D * dm.dd);
        DP_CUDA_TRY(allow_big_smem((const void *)row_prep_kernel, smem));
        row_prep_kernel<<<n, kThreads, smem, st>>>(dm, params, rows, rpc, adv, p->act_p, p->act_choice, p->act_u,
                                                 p->act_h, p->act_ctx, p->row_q, p->row_dctx, p->row_w, p->row_dhx,
                                                 part);
        DP_LAUNCH_CHECK();
        const int na = dm.D + dm.D * dm.dd + 2 * kH * dm.dd;
        // [b_out | dev[:D] | w_out]
        reduce_partials_kernel<<<ceil_div(dm.D, 256), 256, 0, st>>>(part, n, na, dm.D, grad + dm.off.b_out, 0);
        reduce_partials_kernel<<<ceil_div(dm.D * dm.dd, 256), 256, 0, st>>>(part + dm.D, n, na, dm.D * dm.dd,
                                                                            grad + dm.off.dev_table, 0);
        reduce_partials_kernel<<<ceil_div(2 * kH * dm.dd, 256), 256, 0, st>>>(
            part + dm.D + dm.D * dm.dd, n, na, 2 * kH * dm.dd, grad + dm.off.w_out, 0);
        DP_LAUNCH_CHECK();
    }
    // B1
    {
        const int n_tiles = ceil_div(rows, kTile);
        const int n = n_cta_for(n_tiles, 2);
        const int tpc = ceil_div(n_tiles, n);
        const int n_used = ceil_div(n_tiles, tpc);
        const size_t smem = sizeof(AttSmem);
        DP_CUDA_TRY(allow_big_smem((const void *)att_bwd_kernel, smem));
        att_bwd_kernel<<<n_used, kThreads, smem, st>>>(dm, rows, tpc, p->enc_h, p->act_stat, p->row_q, p->row_dctx,
                                                       p->row_w, p->row_dq, part);
        DP_LAUNCH_CHECK();
        reduce_partials_kernel<<<ceil_div(T * kH, 256), 256, 0, st>>>(part, n_used, (size_t)T * kH, T * kH,
                                                                      p->d_enc, 0);
        DP_LAUNCH_CHECK();
    }
    // B1f
    {
        const int n = n_cta_for(rows, 64);
        const int rpc = ceil_div(rows, n);
        row_fin_kernel<<<n, kThreads, 0, st>>>(dm, params, rows, rpc, p->act_h, p->row_dq, p->row_dhx, part);
        DP_LAUNCH_CHECK();
        reduce_partials_kernel<<<ceil_div(kH * kH, 256), 256, 0, st>>>(part, n, kH * kH, kH * kH,
                                                                       grad + dm.off.w_att, 0);
        DP_LAUNCH_CHECK();
    }
    // B2: decoder LSTM backward, per sample
    {
        int M = ceil_div(K, kNumSMs);
        if (M > 8) M = 8;
        const size_t smem = sizeof(double) * (size_t)M * (2 * kH + kG);
        DP_CUDA_TRY(allow_big_smem((const void *)lstm_bwd_kernel, smem));
        lstm_bwd_kernel<<<ceil_div(K, M), kThreads, smem, st>>>(
            T, K, M, params + dm.off.w_dec + (size_t)dm.dd * kG, p->act_g, p->act_c, p->enc_c + (size_t)(T - 1) * kH,
            p->row_dhx, nullptr, nullptr, p->dh0, p->dc0);
        DP_LAUNCH_CHECK();
    }
    // B3
    {
        const int n = n_cta_for(rows, 128);
        const int rpc = ceil_div(rows, n);
        const size_t smem = sizeof(double) * (dm.D + 1) * kG;
        DP_CUDA_TRY(allow_big_smem((const void *)dec_wgrad_kernel, smem + 32 * 1024));
        dec_wgrad_kernel<<<n, kThreads, smem, st>>>(dm, rows, rpc, p->act_h, p->enc_h, p->act_choice, p->act_g,
                                                    part);
        DP_LAUNCH_CHECK();
        const size_t stride = (size_t)(kH + dm.D + 1) * kG;
        reduce_partials_kernel<<<ceil_div(kH * kG, 256), 256, 0, st>>>(part, n, stride, kH * kG,
                                                                       grad + dm.off.w_dec + (size_t)dm.dd * kG, 0);
        reduce_partials_kernel<<<ceil_div((dm.D + 1) * kG, 256), 256, 0, st>>>(part + (size_t)kH * kG, n, stride,
                                                                               (dm.D + 1) * kG, p->gacc, 0);
        DP_LAUNCH_CHECK();
        dec_finalize_kernel<<<1, kG, 0, st>>>(dm, params, p->gacc, grad);
        DP_LAUNCH_CHECK();
    }
    // B4: encoder backward once on the summed inputs
    {
        sum_rows_kernel<<<1, kH, 0, st>>>(p->dh0, K, dhc_sum);
        sum_rows_kernel<<<1, kH, 0, st>>>(p->dc0, K, dhc_sum + kH);
        DP_LAUNCH_CHECK();
        DP_CUDA_TRY(cudaMemcpyAsync(p->da_enc, p->enc_g, sizeof(double) * T * kG, cudaMemcpyDeviceToDevice, st));
        const size_t smem = sizeof(double) * (2 * kH + kG);
        lstm_bwd_kernel<<<1, kThreads, smem, st>>>(T, 1, 1, params + dm.off.w_enc + (size_t)dm.F * kG, p->da_enc,
                                                   p->enc_c, p->zeros, p->d_enc, dhc_sum, dhc_sum + kH,
                                                   p->dh0, p->dc0);
        DP_LAUNCH_CHECK();
    }
    // B5
    {
        enc_wgrad_kernel<<<dm.F + kH + 1, kG, 0, st>>>(dm, p->X, p->enc_h, p->da_enc, grad);
        DP_LAUNCH_CHECK();
        enc_dx_kernel<<<ceil_div(T * dm.td, 256), 256, 0, st>>>(dm, params, p->da_enc, dx_scratch);
        DP_LAUNCH_CHECK();
        type_scatter_kernel<<<ceil_div(dm.V1 * dm.td, 128), 128, 0, st>>>(dm, p->occ_off, p->occ_t, p->type_off,
                                                                          dx_scratch, grad);
        DP_LAUNCH_CHECK();
    }
    return DP_OK;
}
