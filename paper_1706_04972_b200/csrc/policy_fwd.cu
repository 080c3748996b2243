// Policy forward on sm_100a: encoder (once per parameter snapshot) and the
// attentional decoder that samples K placements at once.
//
// Reference: /root/reference/pkg/src/devplace/policy.py
//   inputs      _assemble_inputs        policy.py:256-263
//   LSTM cell   _lstm_step / _sigmoid   policy.py:220-233  (gate order i, f, o, g)
//   encoder     _forward                policy.py:276-287
//   decoder     _forward                policy.py:288-311
//   sampling    forward_sample.choose   policy.py:317-326
//
// Everything is IEEE fp64 like the reference (numpy float64): sampled indices
// must be bit-exact, and fp32/TF32 flip 0.006-1.2 draws per update
// (SURVEY.md §0.5).  Design:
//   * the encoder is identical for all K samples, so it runs ONCE per snapshot
//     (the reference reruns it per sample): x@W_x+b for all t is one parallel
//     GEMM, only h@W_h (64x256) stays sequential — one CTA, one thread per gate
//     column with its 64 W_h weights in registers, 4 gates of a unit in 4
//     adjacent lanes (shuffle exchange, one barrier per step);
//   * the decoder input projection collapses to a (D+1)x256 table
//     edev = dev_table @ W_dec[:dd] + b_dec, gathered by the previous choice;
//   * attention uses s = enc @ (W_att^T h) (== (enc @ W_att^T) @ h, the
//     reference's proj @ h) so only enc_states (T x 64) is needed; it is staged
//     in shared memory with a padded stride (conflict-free for both the
//     row-per-thread score pass and the column-per-lane context pass);
//   * one CTA owns M samples for all T steps (samples are independent, no grid
//     sync); the softmax / PCG64 draw / log-prob tail runs warp-per-sample.

#include <math.h>

#include <vector>

#include "cpasync.cuh"
#include "fastmath.cuh"
#include "pcg64.cuh"
#include "policy.cuh"
#include "tc.cuh"

namespace dp {

__device__ __forceinline__ double sigmoid_ref(double x) { return 1.0 / (1.0 + exp(-x)); }

// LSTM gate activation without warp divergence between the sigmoid gates and
// the tanh gate: both go through ONE expm1 and one division,
//   sigmoid(x) = 1 / (2 + expm1(-x)),
//   tanh(x)    = sign(x) * (-e / (2 + e)),  e = expm1(-2|x|)  (e in (-1, 0]).
// expm1 keeps tanh's relative accuracy near 0 and nothing overflows; the
// result differs from numpy's 1/(1+exp(-x)) / tanh(x) by ~1 ulp (same order
// as the dot-product summation-order differences).
// The expm1 and the division are the branch-free fastmath.cuh versions, so the
// activations of a thread's M samples overlap (libm's slow-path branches
// serialise them).
__device__ __forceinline__ double gate_act(double x, bool is_tanh) { return fm_gate_act(x, is_tanh); }
__device__ __forceinline__ double tanh_x(double x) { return gate_act(x, true); }

// Debug-only per-phase cycle counters of the decoder (block 0, thread 0).
__device__ int g_dbg_clocks = 0;
__device__ long long g_phase_clk[16];
__device__ long long g_warp_clk[8 * 3];
// debug: per-warp phase-end arrival (block 0), summed over steps (g_warp_clk above)
__device__ int g_dbg_skip = 0;  // debug-only ablation bits (timing experiments; results invalid when set)

// numpy pairwise_sum order for n <= 128 (np.add.reduce on a contiguous array):
// n < 8 sequential; otherwise 8 interleaved accumulators, fixed tree, tail.
__device__ __forceinline__ double np_sum_small(const double *a, int n) {
    if (n < 8) {
        double r = 0.0;
        for (int i = 0; i < n; i++) r += a[i];
        return r;
    }
    double r[8];
#pragma unroll
    for (int j = 0; j < 8; j++) r[j] = a[j];
    int i = 8;
    for (; i < n - (n % 8); i += 8) {
#pragma unroll
        for (int j = 0; j < 8; j++) r[j] += a[i + j];
    }
    double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; i++) res += a[i];
    return res;
}

// ---------------------------------------------------------------- prologue
// One launch for the encoder prologue.  Blocks t < T: the input row
//   X[t] = [mean(type_table[idx_t]) | shape_t | adj_t]   (policy.py:256-263)
// (kept in X for the w_enc gradient) and its gate pre-activation
//   XP[t] = X[t] W_enc[:F] + b_enc;
// blocks T .. T+D: edev[d] = dev_table[d] W_dec[:dd] + b_dec (d = D: the start
// row, dev_table[D]).  Thread j owns gate column j; 4 accumulators keep the
// weight loads in flight.
__global__ void __launch_bounds__(kG) enc_prologue_kernel(PolicyDims dm, const double *__restrict__ params,
                                                          const int32_t *__restrict__ type_off,
                                                          const int32_t *__restrict__ type_idx,
                                                          const double *__restrict__ shape,
                                                          const double *__restrict__ adj, double *__restrict__ X,
                                                          double *__restrict__ XP, double *__restrict__ edev) {
    __shared__ double xs[512];
    const int j = threadIdx.x;
    const bool enc = blockIdx.x < dm.T;
    const int t = blockIdx.x, d = blockIdx.x - dm.T;
    const int K = enc ? dm.F : dm.dd;
    if (enc) {
        for (int f = j; f < dm.F; f += kG) {
            double v;
            if (f < dm.td) {
                // numpy mean(axis=0): first row, then sequential adds, then / count
                const double *tab = params + dm.off.type_table;
                const int a = type_off[t], b = type_off[t + 1];
                double s = tab[(size_t)type_idx[a] * dm.td + f];
                for (int i = a + 1; i < b; i++) s = s + tab[(size_t)type_idx[i] * dm.td + f];
                v = s / (double)(b - a);
            } else if (f < dm.td + dm.ss) {
                v = shape[(size_t)t * dm.ss + (f - dm.td)];
            } else {
                v = adj[(size_t)t * dm.as + (f - dm.td - dm.ss)];
            }
            xs[f] = v;
            X[(size_t)t * dm.F + f] = v;
        }
    } else {
        for (int o = j; o < dm.dd; o += kG) xs[o] = params[dm.off.dev_table + (size_t)d * dm.dd + o];
    }
    __syncthreads();
    const double *W = params + (enc ? dm.off.w_enc : dm.off.w_dec) + j;
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    int i = 0;
    for (; i + 4 <= K; i += 4) {
        a0 = fma(xs[i], W[(size_t)i * kG], a0);
        a1 = fma(xs[i + 1], W[(size_t)(i + 1) * kG], a1);
        a2 = fma(xs[i + 2], W[(size_t)(i + 2) * kG], a2);
        a3 = fma(xs[i + 3], W[(size_t)(i + 3) * kG], a3);
    }
    for (; i < K; i++) a0 = fma(xs[i], W[(size_t)i * kG], a0);
    const double v = ((a0 + a1) + (a2 + a3)) + params[(enc ? dm.off.b_enc : dm.off.b_dec) + j];
    if (enc) XP[(size_t)t * kG + j] = v;
    else edev[(size_t)d * kG + j] = v;
}

// mma.sync m8n8k4 f64 (DMMA): D[8x8] += A[8x4] B[4x8], one warp; lane = 4 g + t:
// a = A[g][t], b = B[t][g], d = {D[g][2t], D[g][2t+1]}
__device__ __forceinline__ void dmma_f64(double (&d)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d[0]), "+d"(d[1])
                 : "d"(a), "d"(b));
}

// 64-term dot of a shared-memory vector (broadcast) with a register column.
__device__ __forceinline__ double dot64_sh_reg(const double *__restrict__ hs, const double (&w)[kH]) {
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
#pragma unroll
    for (int k = 0; k < kH; k += 4) {
        const double2 h01 = *reinterpret_cast<const double2 *>(hs + k);
        const double2 h23 = *reinterpret_cast<const double2 *>(hs + k + 2);
        a0 = fma(h01.x, w[k], a0);
        a1 = fma(h01.y, w[k + 1], a1);
        a2 = fma(h23.x, w[k + 2], a2);
        a3 = fma(h23.y, w[k + 3], a3);
    }
    return (a0 + a1) + (a2 + a3);
}

// ---------------------------------------------------------------- encoder
// One CTA, 256 threads: thread (u, q) = (tid>>2, tid&3) holds unit u's four
// gate columns of W_enc's h-rows for the input quarter k in [16q, 16q+16) in
// registers.  Per step: 8 h loads (the warp's 4 quarters are 4 distinct
// addresses per load, not a 64-value broadcast per lane), 4 partial dots, a
// 4-lane reduce-scatter that leaves gate q's full pre-activation in lane q
// (= the gate column col = q*64 + u), activation, 4-lane shuffle to the
// unit's owner, c/h update, one barrier.
// CLK: debug phase clocks compiled in (a separate instantiation: disabled
// instrumentation still costs issue slots on this latency-bound chain)
template <bool CLK>
__global__ void __launch_bounds__(kThreads, 1)
    enc_rec_kernel(PolicyDims dm, const double *__restrict__ params, const double *__restrict__ XP,
                   double *__restrict__ enc_h, double *__restrict__ enc_c, double *__restrict__ enc_g) {
    __shared__ __align__(16) double hbuf[2][kH + 8];  // quarter q at 18q: conflict-free
    const int tid = threadIdx.x, lane = tid & 31;
    const int u = tid >> 2, gate = tid & 3, col = gate * kH + u;
    const double *Wh = params + dm.off.w_enc + (size_t)dm.F * kG;
    double w[4][16];
#pragma unroll
    for (int g = 0; g < 4; g++)
#pragma unroll
        for (int k = 0; k < 16; k++) w[g][k] = Wh[(size_t)(16 * gate + k) * kG + g * kH + u];
    if (tid < kH + 8) hbuf[0][tid] = 0.0;
    double c = 0.0;
    // XP two steps ahead in registers (a step is ~1.4K cycles, an L2/HBM load can take most of one)
    double xp = dm.T > 0 ? XP[col] : 0.0, xp2 = dm.T > 1 ? XP[kG + col] : 0.0;
    __syncthreads();
    const int base = lane & ~3;
    const bool hi = gate & 2, lo = gate & 1;
    const bool clk_on = CLK && tid == 0;  // debug phase clocks -> g_phase_clk[4..7]
    long long ck[4] = {0, 0, 0, 0}, c_last = clk_on ? clock64() : 0;
#define DP_ENC_PHASE(i)                      \
    if (clk_on) {                            \
        const long long now_ = clock64();    \
        ck[i] += now_ - c_last;              \
        c_last = now_;                       \
    }
    for (int t = 0; t < dm.T; t++) {
        const double2 *hq = reinterpret_cast<const double2 *>(hbuf[t & 1] + 18 * gate);
        double p[4][2];
#pragma unroll
        for (int g = 0; g < 4; g++) p[g][0] = p[g][1] = 0.0;
#pragma unroll
        for (int k = 0; k < 8; k++) {
            const double2 hv = hq[k];
#pragma unroll
            for (int g = 0; g < 4; g++) {
                p[g][0] = fma(hv.x, w[g][2 * k], p[g][0]);
                p[g][1] = fma(hv.y, w[g][2 * k + 1], p[g][1]);
            }
        }
        const double p0 = p[0][0] + p[0][1], p1 = p[1][0] + p[1][1];
        const double p2 = p[2][0] + p[2][1], p3 = p[3][0] + p[3][1];
        // reduce-scatter over the 4 quarter lanes: lane q ends with gate q's sum
        double k0 = hi ? p2 : p0, k1 = hi ? p3 : p1;
        k0 += __shfl_xor_sync(0xffffffffu, hi ? p0 : p2, 2);
        k1 += __shfl_xor_sync(0xffffffffu, hi ? p1 : p3, 2);
        double kk = lo ? k1 : k0;
        kk += __shfl_xor_sync(0xffffffffu, lo ? k0 : k1, 1);
        const double a = xp + kk;
        DP_ENC_PHASE(0);
        xp = xp2;
        if (t + 2 < dm.T) xp2 = XP[(size_t)(t + 2) * kG + col];
        const double act = fm_gate_act<true>(a, gate == 3);  // constant-bank coefficients (measured faster here)
        DP_ENC_PHASE(1);
        enc_g[(size_t)t * kG + col] = act;
        const double iv = __shfl_sync(0xffffffffu, act, base + 0);
        const double fv = __shfl_sync(0xffffffffu, act, base + 1);
        const double ov = __shfl_sync(0xffffffffu, act, base + 2);
        const double gv = __shfl_sync(0xffffffffu, act, base + 3);
        if (gate == 0) {
            c = fv * c + iv * gv;
            const double h = ov * fm_gate_act<true>(c, true);
            hbuf[(t + 1) & 1][u + 2 * (u >> 4)] = h;
            enc_h[(size_t)t * kH + u] = h;
            enc_c[(size_t)t * kH + u] = c;
        }
        DP_ENC_PHASE(2);
        __syncthreads();
        DP_ENC_PHASE(3);
    }
#undef DP_ENC_PHASE
    if (clk_on)
        for (int i = 0; i < 4; i++) g_phase_clk[4 + i] += ck[i];
}

// Encoder recurrence on a cluster of kEncCl CTAs (opt-in, dp_debug_encoder_variant(1);
// measured slower: 2.2K vs 1.4K cycles per step).  CTA r owns units
// [16 r, 16 r + 16), i.e. 64 of the 256 gate columns, so each SM issues a quarter
// of the step's h W_h FMAs (the one-CTA kernel above is bound by the SM's fp64
// pipe in that phase).  Thread lane = (u2, gate, kq): 4 lanes split a column's k
// range (16 W_h values each in registers), two xor shuffles give every lane the
// full pre-activation; the unit's 16 lanes gather i / f / o / g and update c
// redundantly, and one lane per unit stores h_t into the step-parity h buffer of
// every CTA of the cluster with st.async (DSMEM), which completes 8 bytes of that
// CTA's buffer mbarrier transaction count (thread 0 of each CTA arms it with the
// 64 values' bytes).  Every thread waits on its own CTA's barrier before the next
// step's dot products: no CTA-wide barrier inside the loop.  Two buffers suffice:
// a unit's h_t can only be formed after every warp of every CTA has finished the
// step t-1 dot products that read the buffer h_t overwrites.
constexpr int kEncCl = 4;
__device__ __forceinline__ uint32_t cl_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t cl_mapa(const void *p, uint32_t cta) {
    uint32_t a = (uint32_t)__cvta_generic_to_shared(p), r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(cta));
    return r;
}
__device__ __forceinline__ void cl_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__global__ void __cluster_dims__(kEncCl, 1, 1) __launch_bounds__(kThreads, 1)
    enc_rec_cluster_kernel(PolicyDims dm, const double *__restrict__ params, const double *__restrict__ XP,
                           double *__restrict__ enc_h, double *__restrict__ enc_c, double *__restrict__ enc_g) {
    __shared__ __align__(16) double hbuf[2][kH];  // h of the previous step, by step parity
    __shared__ __align__(8) unsigned long long hbar[2];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t rank = cl_rank();
    const int u2 = lane >> 4, gate = (lane >> 2) & 3, kq = lane & 3;
    const int u = (int)rank * 16 + warp * 2 + u2, col = gate * kH + u;
    const double *Wh = params + dm.off.w_enc + (size_t)dm.F * kG;
    double w[16];
#pragma unroll
    for (int k = 0; k < 16; k++) w[k] = Wh[(size_t)(16 * kq + k) * kG + col];
    if (tid < kH) hbuf[0][tid] = 0.0;
    // one local arrival per phase (thread 0's expect_tx of the 64 h values' bytes);
    // the values themselves complete the transaction count (st.async)
    const uint32_t hb0 = (uint32_t)__cvta_generic_to_shared(&hbar[0]);
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(hb0) : "memory");
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(hb0 + 8) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    double c = 0.0;
    double xp = dm.T > 0 ? XP[col] : 0.0, xp2 = dm.T > 1 ? XP[kG + col] : 0.0;
    const int base = lane & 16;
    const bool writer = gate == 0 && kq == 0;
    // cluster addresses of h[u] and of the barriers (buffer 0) in every CTA; buffer 1
    // is at the same offset in each CTA's window
    uint32_t rh[kEncCl], rb[kEncCl];
#pragma unroll
    for (int q = 0; q < kEncCl; q++) {
        rh[q] = cl_mapa(&hbuf[0][u], q);
        rb[q] = cl_mapa(&hbar[0], q);
    }
    constexpr uint32_t kHOff = kH * sizeof(double), kBOff = sizeof(unsigned long long);
    cl_sync();  // barriers initialised and h_{-1} zeroed in every CTA before any remote access
    for (int t = 0; t < dm.T; t++) {
        const int b = t & 1;
        if (t > 0) {
            // h_{t-1} complete in this CTA (buffer b's phase (t-1)/2)
            const uint32_t par = (uint32_t)((t - 1) >> 1) & 1u;
            asm volatile(
                "{\n"
                ".reg .pred p;\n"
                "DP_ENC_WAIT_%=:\n"
                "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
                "@!p bra DP_ENC_WAIT_%=;\n"
                "}\n" ::"r"(hb0 + 8u * (uint32_t)b),
                "r"(par)
                : "memory");
        }
        // arm the buffer h_t lands in (its previous phase, h_{t-2}, completed before
        // this thread's wait at step t-1)
        if (tid == 0 && t + 1 < dm.T)
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(hb0 + 8u * (uint32_t)(b ^ 1)),
                         "r"((uint32_t)(kH * sizeof(double)))
                         : "memory");
        const double2 *hq = reinterpret_cast<const double2 *>(hbuf[b] + 16 * kq);
        double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
#pragma unroll
        for (int k = 0; k < 8; k += 2) {
            const double2 h0 = hq[k], h1 = hq[k + 1];
            a0 = fma(h0.x, w[2 * k], a0);
            a1 = fma(h0.y, w[2 * k + 1], a1);
            a2 = fma(h1.x, w[2 * k + 2], a2);
            a3 = fma(h1.y, w[2 * k + 3], a3);
        }
        double pre = (a0 + a1) + (a2 + a3);
        pre += __shfl_xor_sync(0xffffffffu, pre, 1);
        pre += __shfl_xor_sync(0xffffffffu, pre, 2);
        const double act = fm_gate_act<true>(xp + pre, gate == 3);
        xp = xp2;
        if (t + 2 < dm.T) xp2 = XP[(size_t)(t + 2) * kG + col];
        if (kq == 0) enc_g[(size_t)t * kG + col] = act;
        const double iv = __shfl_sync(0xffffffffu, act, base + 0);
        const double fv = __shfl_sync(0xffffffffu, act, base + 4);
        const double ov = __shfl_sync(0xffffffffu, act, base + 8);
        const double gv = __shfl_sync(0xffffffffu, act, base + 12);
        c = fv * c + iv * gv;
        if (writer) {
            const double h = ov * fm_gate_act<true>(c, true);
            const uint32_t nb = (uint32_t)(b ^ 1);
            if (t + 1 < dm.T)
#pragma unroll
                for (int q = 0; q < kEncCl; q++)
                    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];" ::"r"(
                                     rh[q] + nb * kHOff),
                                 "d"(h), "r"(rb[q] + nb * kBOff)
                                 : "memory");
            enc_h[(size_t)t * kH + u] = h;
            enc_c[(size_t)t * kH + u] = c;
        }
    }
    cl_sync();  // no CTA leaves while a peer may still write into its shared memory
}

// ---------------------------------------------------------------- decoder
// Per-snapshot decoder prologue, shared by all K samples (once per update):
//   proj = enc_states @ W_att^T    [T x 64]  (policy.py:287 — the reference's own order)
//   encW = enc_states @ W_out[64:] [T x dd]  (ctx @ W_out[64:] == alpha @ encW, so the
//                                            step's context never has to be formed)
// Also: proj_nmax = max_t ||proj_t||_2 (atomic max on the IEEE bits of a
// non-negative double; zeroed by the caller).  |s_t| = |proj_t . h| <
// 8 ||proj_t|| because |h_j| < 1 (h = o * tanh(c), 64 units), so when
// 8 * proj_nmax <= kNoShiftBound the decoder's softmax over the T scores can
// skip the max subtraction: exp() neither overflows nor underflows, and
// alpha = exp(s) / sum exp(s) equals the reference's exp(s - max) / sum to
// rounding (the shift cancels exactly in real arithmetic).
constexpr double kNoShiftBound = 600.0;

// Block 0 also forms vdev = W_out[:64] @ dev_table[:D]^T [64][D]: the logits'
// h half becomes one 64-term dot per device (zh_d = h . vdev[:, d]).
__global__ void dec_prep_kernel(PolicyDims dm, const double *__restrict__ params, const double *__restrict__ enc_h,
                                double *__restrict__ proj, double *__restrict__ encW,
                                unsigned long long *__restrict__ proj_nmax, double *__restrict__ vdev) {
    __shared__ double e[kH];
    __shared__ double sq[kH];
    const int t = blockIdx.x, tid = threadIdx.x, dd = dm.dd;
    if (tid < kH) e[tid] = enc_h[(size_t)t * kH + tid];
    if (t == 0)
        for (int x = tid; x < kH * dm.D; x += blockDim.x) {
            const int l = x / dm.D, d = x - l * dm.D;
            double v = 0.0;
            for (int o = 0; o < dd; o++)
                v = fma(params[dm.off.w_out + (size_t)l * dd + o], params[dm.off.dev_table + (size_t)d * dd + o], v);
            vdev[x] = v;
        }
    __syncthreads();
    double a0 = 0.0, a1 = 0.0;
    if (tid < kH) {
        const double *w = params + dm.off.w_att + (size_t)tid * kH;  // W_att[l][:]
        for (int j = 0; j < kH; j += 2) {
            a0 = fma(e[j], w[j], a0);
            a1 = fma(e[j + 1], w[j + 1], a1);
        }
        proj[(size_t)t * kH + tid] = a0 + a1;
        sq[tid] = (a0 + a1) * (a0 + a1);
    } else if (tid < kH + dd) {
        const int o = tid - kH;
        const double *w = params + dm.off.w_out + (size_t)kH * dd + o;  // W_out[64 + j][o]
        for (int j = 0; j < kH; j += 2) {
            a0 = fma(e[j], w[(size_t)j * dd], a0);
            a1 = fma(e[j + 1], w[(size_t)(j + 1) * dd], a1);
        }
        encW[(size_t)t * dd + o] = a0 + a1;
    }
    __syncthreads();
    if (tid == 0) {
        double n2 = 0.0;
        for (int l = 0; l < kH; l++) n2 += sq[l];
        atomicMax(proj_nmax, (unsigned long long)__double_as_longlong(sqrt(n2)));
    }
}

constexpr int kProjLd = 66;
constexpr int kWout1Ld = kH + 8;  // W_out[:64]^T row stride (== 8 mod 16 doubles: 8-lane groups in distinct banks)  // proj row stride in shared memory: 16-byte rows, conflict-free LDS.128
constexpr int kWarps = kThreads / 32;
static_assert(kWarps == 8, "g_warp_clk is sized for 8 warps");
// DM streaming (C5-sized T, noshift): per-warp cp.async ring of 8-row blocks of
// proj ([8][64]) and encW ([8][16]), XOR-swizzled by 16-byte chunk so the DMMA
// fragment loads are conflict-free without padding; 4 slots per warp (two
// blocks computed while the next two arrive), aliased onto the score rows alS
constexpr int kDmsSlot = 8 * 64 + 8 * 16, kDmsSlots = 4;
// word offset of proj element (r, k) / encW element (r, j) inside a slot
__device__ __forceinline__ int dms_p(int r, int k) { return r * 64 + 2 * ((k >> 1) ^ r) + (k & 1); }
__device__ __forceinline__ int dms_e(int r, int j) {
    return 8 * 64 + r * 16 + 2 * ((j >> 1) ^ (((r >> 1) & 1) << 2)) + (j & 1);
}

// sum_w fw[w] p[w * stride] over the 8 warp partials as a tree (depth 4)
__device__ __forceinline__ double wsum8(const double *p, int stride, const double (&fw)[kWarps]) {
    const double a = fma(p[stride], fw[1], p[0] * fw[0]);
    const double b = fma(p[3 * stride], fw[3], p[2 * stride] * fw[2]);
    const double c = fma(p[5 * stride], fw[5], p[4 * stride] * fw[4]);
    const double d = fma(p[7 * stride], fw[7], p[6 * stride] * fw[6]);
    return (a + b) + (c + d);
}


struct DecArgs {
    PolicyDims dm;
    const double *params;
    int K;
    long long k_offset;
    uint64_t st_hi, st_lo, inc_hi, inc_lo;
    unsigned long long draw_base;
    const long long *draw_counter;
    long long draws_per_count;
    const uint8_t *forced;
    const double *enc_h, *enc_c, *edev, *proj, *encW;
    const unsigned long long *proj_nmax;
    const double *vdev;
    double *act_h, *act_c, *act_g, *act_uc, *act_u, *act_p, *act_stat, *act_lz, *act_e, *act_esc;
    uint8_t *choice, *choice_out;
    double *logp, *probs_out;
    double *margin;  // [K] or NULL: min over steps of min_{j<D-1} |r - cdf_j| (sampling only)
    int M, Tpad, ewld;
    // shared-memory offsets (doubles)
    int o_proj, o_encw, o_wout, o_devt, o_bout, o_edev, o_h, o_uh, o_alpha, o_pm, o_ps, o_puc, o_pz, o_gn, o_hc,
        o_cc, o_ac, o_pcg, o_misc, o_v, o_wo, o_rn, o_fin;
    int o_bdig, o_tmb;  // TCG: h digit-plane stacks (B operands), mbarrier + TMEM base
};

// q = x / n for 0 <= x < MT * n without an integer division (MT <= 8)
template <int MT>
__device__ __forceinline__ int small_div(int x, int n) {
    int q = 0;
#pragma unroll
    for (int k = 1; k < MT; k++) q += x >= k * n ? 1 : 0;
    return q;
}

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// One CTA owns M samples for all T decode steps.  Per step:
//   [A] (non-speculative variant only) gates = edev[prev] + g, LSTM cell -> h
//   C   (all warps) fused pass: s_i = proj_i . h for the thread's rows and the
//       next step's g = h W_h for its gate column (shared h loads); warp-local
//       softmax statistics (max m_w, sum l_w), partial uc_w = sum_i e_i encW_i
//       and partial logits pz_w = dev_table[:D] uc_w; uh = h W_out[:64]
//   E   warp per sample: online-softmax combine of the 8 warp partials
//       (M = max m_w, l = sum l_w e^{m_w-M}), z = dev_table[:D] uh + b_out +
//       (sum_w pz_w e^{m_w-M}) / l, softmax over devices, PCG64 draw, cdf search.
//       SPEC: the idle warps meanwhile evaluate the next step's LSTM cell for
//       every possible choice d (edev[d] + g), so the next step starts at C
//       with h = candidate[choice] and phase A disappears from the chain.
// The context vector is never formed: ctx @ W_out[64:] = alpha @ encW, and the
// backward works from uc (w = uc.du, dW_out[64:] = enc^T sum alpha^T du).
// FAST (MT <= 2, D <= 4, dd <= 16, T <= 256, proj in shared memory, no SPEC):
// the generic alternatives are compiled out, so the per-step loop's hot code
// is compact (the draw chain measurably stalls on instruction fetch when it
// jumps across the cold paths).
// FAST: the draw warp leaves step s's (esum, gmx, gsum, zs[D], ez[D]) in fin
// and its choice in prev; a pcg warp finishes the row one step later, off the
// draw chain: the probabilities p = ez / esum, the row's global cache entries,
// and the sampling margin min_j<D-1 |r - cdf_j| with cdf = cumsum(p) (the
// reference's searchsorted(cumsum(p), r), pkg/policy.py:320-323) against the
// step's uniform r (still in rnext: the caller runs this before the pcg step
// that overwrites it).
template <int FS = 16, int EZO = 8>  // record stride and the ez offset (D <= 4: 16 / 8; D <= 8: 24 / 12)
__device__ __forceinline__ void fin_store(const DecArgs &a, double *fin, const int *prev, const double *rnext,
                                          int k0, int m, int M, int T, int s) {
    if (k0 + m >= a.K) return;
    const int D = a.dm.D;
    const size_t row = (size_t)(k0 + m) * T + s;
    const int ch = prev[(((s & 1) ^ 1) * M) + m];
    const double *f = fin + ((s & 1) * M + m) * FS;
    const double esum = f[0];
    const double y = fm_rcp(esum);
    const double r = rnext[(s & 1) * M + m];
    double cdf = 0.0, mg = INFINITY;
    for (int d = 0; d < D; d++) {
        const double p = fm_div_y(f[EZO + d], esum, y);
        a.act_p[row * D + d] = p;
        if (a.probs_out) a.probs_out[row * D + d] = p;
        cdf += p;
        if (d < D - 1) mg = fmin(mg, fabs(r - cdf));
    }
    a.choice[row] = (uint8_t)ch;
    if (a.choice_out) a.choice_out[row] = (uint8_t)ch;
    a.act_lz[row * 2] = f[4 + ch];
    a.act_lz[row * 2 + 1] = esum;
    a.act_stat[row * 2] = f[1];  // softmax stats (max, sum) for the backward's recompute of alpha
    a.act_stat[row * 2 + 1] = f[2];
    if (!a.forced) fin[2 * FS * M + m] = fmin(fin[2 * FS * M + m], mg);
}

template <int MT, bool PS, bool SPEC, bool FAST = false, bool TCG = false, bool CLK = false, int DX = 4>
__global__ void __launch_bounds__(kThreads, 1) dec_kernel(DecArgs a) {
    static_assert(DX == 4 || (DX == 8 && FAST), "DX: the FAST path's device bound (4 or 8)");
    // FAST draw layout: NP lanes per device in the logits, the step record stride FS and
    // the ez offset EZO in it (D <= 4: 8 / 16 / 8; D <= 8: 4 / 24 / 12)
    constexpr int NP = DX == 8 ? 4 : 8, FS = DX == 8 ? 24 : 16, EZO = 4 + DX;
    static_assert(!TCG || (FAST && PS && !SPEC && MT <= 2), "TCG is a FAST-path variant");
    extern __shared__ __align__(16) double sm[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const PolicyDims &dm = a.dm;
    const int T = dm.T, D = dm.D, dd = dm.dd, M = a.M;
    const int k0 = blockIdx.x * M;
    const int Mb = min(M, a.K - k0);
    const double *P = a.params;
    constexpr int LD = PS ? kProjLd : kH;
    const double *proj = PS ? (const double *)(sm + a.o_proj) : a.proj;
    const double *encW = PS ? (const double *)(sm + a.o_encw) : a.encW;
    double *wout1 = sm + a.o_wout;  // W_out[:64]^T [dd][kWout1Ld]
    double *devt = sm + a.o_devt;
    double *bout = sm + a.o_bout;
    double *edevS = sm + a.o_edev;  // (non-SPEC) edev staged
    double *hS = sm + a.o_h;        // (non-SPEC) [M][64]
    double *uhS = sm + a.o_uh;      // [M][32]
    double *alS = sm + a.o_alpha;   // [M][Tpad] scores -> e_i
    double *pmx = sm + a.o_pm;      // [8][M] warp max
    double *psm = sm + a.o_ps;      // [8][M] warp sum
    double *puc = sm + a.o_puc;     // [8][M][dd] warp uc partials
    double *pz = sm + a.o_pz;       // [8][M][D] warp partial logits
    double *gnS = sm + a.o_gn;      // (SPEC) [M][256] next step's h W_h
    double *hC = sm + a.o_hc;       // (SPEC) [M][D][64] candidate h
    double *cC = sm + a.o_cc;       // (SPEC) [2][M][D][64] candidate c (step parity)
    double *aC = sm + a.o_ac;       // (SPEC) [M][D][256] candidate gate activations
    unsigned long long *pcg = reinterpret_cast<unsigned long long *>(sm + a.o_pcg);  // [M][2]
    int *prev = reinterpret_cast<int *>(sm + a.o_misc);  // [2][M] previous choice, by step parity
    double *rnext = sm + a.o_rn;  // [2][M] the step's uniform, by step parity (pcg warps)
    double *fin = sm + a.o_fin;   // FAST: [2][M][16] (esum, gmx, gsum, -, zs[4], ez[4]) of the step, by parity; [M] margins
    // pcg warps: with 3 Mb <= 8 warps, warp 8 - Mb + m steps sample m's PCG64 stream
    // during E and leaves the next step's uniform in rnext (off the draw chain)
    const bool pcgw = FAST || 3 * Mb <= kWarps;
    const double *edev = SPEC ? a.edev : edevS;
    // softmax over the T scores without the max shift when |s| is provably small
    const bool noshift = 8.0 * __longlong_as_double((long long)*a.proj_nmax) <= kNoShiftBound;

    // ---- stage the snapshot-constant operands ----
    if (PS) {
        if (!TCG)  // TCG: each thread keeps its proj row in registers instead
            for (int i = tid; i < T * kH; i += kThreads) sm[a.o_proj + (i >> 6) * kProjLd + (i & 63)] = a.proj[i];
        // transposed: encWT[j][i], row stride a.ewld (== 2 mod 32 words apart per j:
        // conflict-free LDS.128 for 8 consecutive j)
        for (int i = tid; i < T * dd; i += kThreads) sm[a.o_encw + (i % dd) * a.ewld + i / dd] = a.encW[i];
    }
    for (int i = tid; i < kH * dd; i += kThreads) wout1[(i % dd) * kWout1Ld + i / dd] = P[dm.off.w_out + i];
    for (int i = tid; i < D * dd; i += kThreads) devt[i] = P[dm.off.dev_table + i];
    double *vS = sm + a.o_v;    // vdev [64][D]
    double *woS = sm + a.o_wo;  // W_out[:64] [64][dd] (row-major: lanes o read consecutive words)
    for (int i = tid; i < kH * D; i += kThreads) vS[i] = a.vdev[i];
    for (int i = tid; i < kH * dd; i += kThreads) woS[i] = P[dm.off.w_out + i];
    for (int i = tid; i < D; i += kThreads) bout[i] = P[dm.off.b_out + i];
    if (!SPEC)
        for (int i = tid; i < (D + 1) * kG; i += kThreads) edevS[i] = a.edev[i];
    // h_{-1} = encoder final state (SPEC: staged in alS, free until step 0's scores)
    double *h0 = SPEC ? alS : hS;
    for (int i = tid; i < (SPEC ? kH : M * kH); i += kThreads) h0[i] = a.enc_h[(size_t)(T - 1) * kH + (i & 63)];
    // both parity halves, all M slots: the per-sample loops compute unguarded
    // (branch-free, so the samples' chains interleave) and only the stores check Mb
    if (tid < 2 * M) prev[tid] = SPEC ? 0 : D;  // SPEC: step 0's state lives in candidate slot 0
    if (FAST && tid < M) fin[2 * FS * M + tid] = INFINITY;  // running sampling margins
    if (MT == 8 && !PS && !SPEC && (dd & 1) == 0)  // DM streaming ring (aliases alS): zero pads
        for (int i = tid; i < kWarps * kDmsSlots * kDmsSlot; i += kThreads) alS[i] = 0.0;
    if (tid < Mb) {
        if (!a.forced) {
            const long long kg = a.k_offset + k0 + tid;
            unsigned long long n0 = a.draw_base + (unsigned long long)kg * (unsigned long long)T;
            if (a.draw_counter) n0 += (unsigned long long)(*a.draw_counter) * (unsigned long long)a.draws_per_count;
            u128 s = pcg_jump(u128{a.st_hi, a.st_lo}, u128{a.inc_hi, a.inc_lo}, n0);
            if (FAST || 3 * Mb <= kWarps) {  // pcgw: step 0's uniform up front
                s = pcg_step(s, u128{a.inc_hi, a.inc_lo});
                rnext[tid] = pcg_double(s);
            }
            pcg[2 * tid] = s.hi;
            pcg[2 * tid + 1] = s.lo;
        }
    }
    const int u = tid >> 2, gate = tid & 3, col = gate * kH + u;
    // w: this thread's W_h gate column (the next step's g = h W_h on the fp64 pipe);
    // TCG: this thread's proj row instead (row tid), and h W_h runs on the tensor
    // cores with W_h's digit planes resident in TMEM (below)
    // DMK (the large-T DM instantiation): W_h is read from L1/L2 when the gate
    // column is formed each step (a few hundred cycles of latency on a ~100K-cycle
    // step), which frees its 128 registers for the streaming score loop
    constexpr bool DMK = MT == 8 && !PS && !SPEC;
    const double *Whcol = P + dm.off.w_dec + (size_t)dd * kG + col;
    double w[kH];
    if (TCG) {
        const double *pr = a.proj + (size_t)(tid < T ? tid : T - 1) * kH;
#pragma unroll
        for (int k = 0; k < kH; k++) w[k] = pr[k];
    } else if (!DMK) {
        const double *Wh = P + dm.off.w_dec + (size_t)dd * kG;
#pragma unroll
        for (int k = 0; k < kH; k++) w[k] = Wh[(size_t)k * kG + col];
    }
    // TCG (tensor-core gates): g = h W_h as fp64-exact int8 digit-plane products
    // (tc.cuh) on tcgen05.mma kind::i8.  A = W_h^T digit planes in TMEM, resident
    // for the whole decode: thread tid writes ITS gate column col into TMEM lane
    // tid % 128 of tile tid / 128 (per (tile, 32-deep k step, plane a): 8 columns
    // of 4 bytes) — exactly the lane quarter its warp may access, so in phase A
    // every thread reads its own column's accumulators back.  B = the step's h
    // digit planes, one stack per k step of 8-row blocks (block b = plane b, row
    // m = sample m, blocks 6.. zero): A plane a multiplies the window starting at
    // block 5 - a, so accumulator block j collects diagonal 5 + j of every plane
    // pair (24 MMAs, M=128, N=48, K=32 per step, issued by two idle warps in E;
    // the dropped pairs a + b < 5 are below 2^-45 of max|W| per term, tc.cuh).
    uint64_t *tmbar = reinterpret_cast<uint64_t *>(sm + a.o_tmb);
    uint32_t *tmslot = reinterpret_cast<uint32_t *>(sm + a.o_tmb + 1);
    uint8_t *bdig = reinterpret_cast<uint8_t *>(sm + a.o_bdig);
    uint32_t tm = 0;
    double gsc = 0.0;  // TCG: 2^(40 - s_col - 46), this column's digit scale
    constexpr uint32_t kTmA = 0, kTmD = 192, kTmCols = 512;  // A planes [0, 192), accumulators [192, 288)
    constexpr int kBStack = 11 * 256;                          // bytes per k step: 6 planes + 5 zero blocks
    if (TCG) {
        for (int i = tid; i < 2 * kBStack / 8; i += kThreads) sm[a.o_bdig + i] = 0.0;
        if (warp == 0) tc::tmem_alloc(tmslot, kTmCols);
        if (tid == 0) {
            tc::mbar_init(tmbar, 2);
            tc::fence_mbar_init();
        }
        tc::fence_before();
        __syncthreads();
        tc::fence_after();
        tm = *tmslot;
        const double *Wh = P + dm.off.w_dec + (size_t)dd * kG + col;
        int eb = 0;
        for (int k = 0; k < kH; k++) eb = max(eb, (__double2hiint(Wh[(size_t)k * kG]) >> 20) & 0x7FF);
        const int sh = tc::fix_shift(eb);
        const double scale = tc::pow2(sh);
        gsc = tc::pow2(40 - sh - tc::kFixBits);
        const uint32_t lane_base = tm + ((uint32_t)((warp & 3) * 32) << 16) + kTmA + (uint32_t)(tid >> 7) * 96;
#pragma unroll 1
        for (int ks = 0; ks < 2; ks++) {
            uint32_t pw[6][8];
#pragma unroll
            for (int c = 0; c < 8; c++) {
#pragma unroll
                for (int b = 0; b < 6; b++) pw[b][c] = 0;
#pragma unroll
                for (int by = 0; by < 4; by++) {
                    const unsigned long long d6 = tc::digits6(Wh[(size_t)(ks * 32 + 4 * c + by) * kG], scale);
#pragma unroll
                    for (int b = 0; b < 6; b++) pw[b][c] |= (uint32_t)((d6 >> (8 * b)) & 0xFF) << (8 * by);
                }
            }
#pragma unroll
            for (int b = 0; b < 6; b++) tc::tmem_st8(lane_base + (uint32_t)(ks * 6 + b) * 8, pw[b]);
        }
        tc::tmem_st_wait();
        tc::fence_before();
    }
    const double c_init = a.enc_c[(size_t)(T - 1) * kH + u];
    double cst[MT];  // (non-SPEC) cell state of unit u, sample m: owned by lane m of the quad (MT <= 4), else gate 0
#pragma unroll
    for (int m = 0; m < MT; m++) cst[m] = c_init;
    const int base = lane & ~3;
    __syncthreads();
    // g = h W_h for the first step (identical initial state for every sample)
    double gn[MT];
    {
        double g0;
        if (TCG || DMK) {
            // step 0 on the fp64 pipe (identical for every sample)
            const double *Wh = P + dm.off.w_dec + (size_t)dd * kG + col;
            double q0 = 0.0, q1 = 0.0;
            for (int k = 0; k < kH; k += 2) {
                q0 = fma(h0[k], Wh[(size_t)k * kG], q0);
                q1 = fma(h0[k + 1], Wh[(size_t)(k + 1) * kG], q1);
            }
            g0 = q0 + q1;
        } else {
            g0 = dot64_sh_reg(h0, w);
        }
#pragma unroll
        for (int m = 0; m < MT; m++) gn[m] = g0;
        if (SPEC) {
            // step 0 (prev = start row D) into candidate slot 0 of every sample
            const double act = gate_act(edev[D * kG + col] + g0, gate == 3);
            const double iv = __shfl_sync(0xffffffffu, act, base + 0);
            const double fv = __shfl_sync(0xffffffffu, act, base + 1);
            const double ov = __shfl_sync(0xffffffffu, act, base + 2);
            const double gv = __shfl_sync(0xffffffffu, act, base + 3);
            const double cn = fv * c_init + iv * gv;
            const double hn = gate == 0 ? ov * tanh_x(cn) : 0.0;
            for (int m = 0; m < Mb; m++) {
                aC[(m * D) * kG + col] = act;
                if (gate == 0) {
                    hC[(m * D) * kH + u] = hn;
                    cC[(m * D) * kH + u] = cn;
                }
            }
        }
    }
    __syncthreads();

    int d_pow2 = 1;
    while (d_pow2 < D) d_pow2 <<= 1;
    // debug phase clocks (dp_debug_phase_clocks): block 0, thread 0, after each barrier
    const bool clk_on = CLK && blockIdx.x == 0 && tid == 0;
    long long clk_last = clk_on ? clock64() : 0;
    long long clk_acc[3] = {0, 0, 0};  // in registers; one global write at the end
    // draw warp m (< Mb <= 8 warps) keeps sample m's running sampling margin
    double mrun = INFINITY;
#define DP_PHASE(i)                                       \
    if (clk_on) {                                         \
        const long long now_ = clock64();                 \
        clk_acc[i] += now_ - clk_last;                    \
        clk_last = now_;                                  \
    }
    const int skip = g_dbg_skip;  // debug ablation bits (dp_debug_phase_clocks), read once
    // debug: each warp's arrival at the phase-ending barrier, from the phase start
    const bool wclk = CLK && blockIdx.x == 0 && lane == 0;
    long long wst = wclk ? clock64() : 0, wacc[3] = {0, 0, 0};
#define DP_WEND(i) \
    if (wclk) wacc[i] += clock64() - wst;
#define DP_WSTART() \
    if (wclk) wst = clock64();
    // running row pointers of the step's cached activations (sample m at + m * T rows)
    const size_t sG = (size_t)T * kG, sH = (size_t)T * kH;
    double *actg = a.act_g + (size_t)k0 * sG + col;
    double *acth = a.act_h + (size_t)k0 * sH + u;
    double *actc = a.act_c + (size_t)k0 * sH + u;
    for (int t = 0; t < T; t++, actg += kG, acth += kH, actc += kH) {
        const int par = t & 1;
        const int *prv = prev + par * M;  // choices of step t-1 (SPEC: candidate slots)
        if (!SPEC) {
            // ---- A: gates + LSTM cell (policy.py:292-294, 224-233) ----
            // every sample slot computes (no branches between the chains); stores check Mb
            double act[MT], cn[MT], hn[MT];
            double hkeep = 0.0, ckeep = 0.0;  // (MT <= 4) this lane's sample: cached after the barrier
            if (TCG && t > 0 && !(skip & 32)) {
                // this column's h_{t-1} W_h from the MMAs issued in the previous E: block j
                // of the accumulator holds diagonal 5 + j for sample m at column 8 j + m;
                // sum_j acc_j 256^(5 + j) in two exact int64 thirds (|acc| < 6 * 64 * 2^14)
                tc::mbar_wait(tmbar, (uint32_t)((t - 1) & 1));
                tc::fence_after();
                const uint32_t lb = tm + ((uint32_t)((warp & 3) * 32) << 16) + kTmD + (uint32_t)(tid >> 7) * 48;
                uint32_t acc[6][2];
#pragma unroll
                for (int j = 0; j < 6; j++) tc::tmem_ld2(lb + 8 * j, acc[j]);
                tc::tmem_ld_wait();
                tc::fence_before();
#pragma unroll
                for (int m = 0; m < MT; m++) {
                    const long long lo = (long long)(int)acc[0][m] + ((long long)(int)acc[1][m] << 8) +
                                         ((long long)(int)acc[2][m] << 16);
                    const long long hi = (long long)(int)acc[3][m] + ((long long)(int)acc[4][m] << 8) +
                                         ((long long)(int)acc[5][m] << 16);
                    gn[m] = fma((double)hi, 16777216.0, (double)lo) * gsc;
                }
            }
#pragma unroll
            for (int m = 0; m < MT; m++)
                act[m] = gate_act(edev[prv[m] * kG + col] + gn[m], gate == 3);
#pragma unroll
            for (int m = 0; m < MT; m++)
                if (m < Mb) actg[m * sG] = act[m];
#pragma unroll
            for (int m = 0; m < MT; m++) {
                const double iv = __shfl_sync(0xffffffffu, act[m], base + 0);
                const double fv = __shfl_sync(0xffffffffu, act[m], base + 1);
                const double ov = __shfl_sync(0xffffffffu, act[m], base + 2);
                const double gv = __shfl_sync(0xffffffffu, act[m], base + 3);
                cn[m] = fv * cst[m] + iv * gv;
                act[m] = ov;
            }
            if (MT <= 4) {
                // lane q of the unit's quad finishes sample q: one tanh per lane
                // (cst[m] is current only in lane m, which is the only reader)
                double cq = cn[0], oq = act[0];
#pragma unroll
                for (int m = 1; m < MT; m++)
                    if (gate == m) {
                        cq = cn[m];
                        oq = act[m];
                    }
                const double hq = oq * tanh_x(cq);
#pragma unroll
                for (int m = 0; m < MT; m++)
                    if (gate == m && m < Mb) {
                        cst[m] = cq;
                        hS[m * kH + u] = hq;
                    }
                hkeep = hq;
                ckeep = cq;
                if (TCG && gate < MT && t + 1 < T && !(skip & 64)) {
                    // sample gate's h[u] -> its 6 digits (|h| < 1: fixed scale 2^46),
                    // plane b into block b, row gate, k = u of the k step's stack
                    const unsigned long long d6 = tc::digits6(hq, 70368744177664.0);  // 2^46
                    const int k = u & 31;
                    uint8_t *bq = bdig + (u >> 5) * kBStack + (k >> 4) * 128 + gate * 16 + (k & 15);
#pragma unroll
                    for (int b = 0; b < 6; b++) bq[b * 256] = (uint8_t)(d6 >> (8 * b));
                    tc::fence_async_smem();
                }
            } else {
#pragma unroll
                for (int m = 0; m < MT; m++) hn[m] = act[m] * tanh_x(cn[m]);
#pragma unroll
                for (int m = 0; m < MT; m++)
                    if (m < Mb && gate == 0) {
                        cst[m] = cn[m];
                        hS[m * kH + u] = hn[m];
                        acth[m * sH] = hn[m];
                        actc[m * sH] = cn[m];
                    }
            }
            DP_WEND(0);
            __syncthreads();
            DP_WSTART();
            if (TCG && warp >= 6 && lane == 0 && t + 1 < T && !(skip & 32)) {
                // the next step's h_t W_h: warp 6 + tl issues tile tl's 12 MMAs right after
                // phase A (measured: issued in E they slow the draw warps' shared-memory loads)
                tc::fence_after();
                constexpr uint32_t idesc = tc::idesc_i8_k(128, 48);
                const int tl = warp - 6;
                const uint32_t b0 = tc::smem_u32(bdig);
#pragma unroll
                for (int ks = 0; ks < 2; ks++)
#pragma unroll
                    for (int aa = 0; aa < 6; aa++)
                        tc::mma_i8_ta(tm + kTmD + 48 * tl, tm + kTmA + tl * 96 + (ks * 6 + aa) * 8,
                                      tc::smem_desc(b0 + ks * kBStack + (5 - aa) * 256, 128, 256), idesc,
                                      (ks | aa) ? 1u : 0u);
                tc::mma_commit(tmbar);
            }
            if (MT <= 4 && gate < Mb) {
                // the step's h / c cache rows after the barrier (off A's tail)
                acth[gate * sH] = hkeep;
                actc[gate * sH] = ckeep;
            }
        }
        DP_PHASE(0);
        // ---- C: scores s = proj @ h (policy.py:296), warp-local softmax stats + partials ----
        const double *hcur[MT];
#pragma unroll
        for (int m = 0; m < MT; m++) hcur[m] = SPEC ? hC + (m * D + (m < Mb ? prv[m] : 0)) * kH : hS + m * kH;
        if (SPEC) {
            // the selected candidate becomes step t's cached activations
#pragma unroll
            for (int m = 0; m < MT; m++)
                if (m < Mb) {
                    const size_t row = (size_t)(k0 + m) * T + t;
                    const int slot = m * D + prv[m];
                    a.act_g[row * kG + col] = aC[slot * kG + col];
                    if (tid < kH) {
                        a.act_h[row * kH + tid] = hcur[m][tid];
                        a.act_c[row * kH + tid] = cC[(par * M * D + slot) * kH + tid];
                    }
                }
        }
        double lmx[MT], lsm[MT];
        // FAST (one score row per thread): the row's scores stay in registers for
        // the exponentials (no shared-memory round trip on the chain)
        double sreg[MT];
#pragma unroll
        for (int m = 0; m < MT; m++) {
            lmx[m] = -INFINITY;
            lsm[m] = 0.0;
            sreg[m] = 0.0;
        }
        // DM (8 samples per CTA, proj too large for shared memory: C5-sized T):
        // the scores are fp64 tensor-core tiles, S[i][m] = proj[i] . h[m] with
        // the 8 samples exactly the DMMA n extent; proj streams from L2
        constexpr bool DM = MT == 8 && !PS && !SPEC;
        const bool dms = DM && noshift && (dd % 2 == 0);  // DM streaming (one pass over T, below)
        if (DM) {
            // next step's gate column g = h W_h (the W_h column from L1/L2, DMK)
            double g0[MT], g1[MT];
#pragma unroll
            for (int m = 0; m < MT; m++) g0[m] = g1[m] = 0.0;
#pragma unroll 8
            for (int j2 = 0; j2 < kH / 2; j2++) {
                const double w0 = __ldg(Whcol + (size_t)(2 * j2) * kG), w1 = __ldg(Whcol + (size_t)(2 * j2 + 1) * kG);
#pragma unroll
                for (int m = 0; m < MT; m++) {
                    const double2 hh = reinterpret_cast<const double2 *>(hcur[m])[j2];
                    g0[m] = fma(hh.x, w0, g0[m]);
                    g1[m] = fma(hh.y, w1, g1[m]);
                }
            }
#pragma unroll
            for (int m = 0; m < MT; m++)
                if (m < Mb) gn[m] = g0[m] + g1[m];
            // B fragments (h of sample g, k = 4 ks + t), reused by every row block
            const int fg = lane >> 2, ft = lane & 3;
            double bf[kH / 4];
#pragma unroll
            for (int ks = 0; ks < kH / 4; ks++) bf[ks] = hS[fg * kH + 4 * ks + ft];
            const int nblk = (T + 7) >> 3;
            if (dms) {
                // streaming (shift-free softmax): each warp owns row blocks warp + 8 k;
                // their proj / encW rows arrive through a 4-slot cp.async ring, two
                // blocks computed per iteration while the next two land.  Per block the
                // warp forms S^T = h proj^T (DMMA, M = the 8 samples, A = h from
                // registers), e = exp(S) in place, the uc partial += e encW (DMMA, A =
                // e straight from the score fragments: k step e' covers rows 2 t + e')
                // and the softmax partial sum — no score rows in shared memory, no
                // barrier, no second pass over T
                double *ring = alS + warp * kDmsSlots * kDmsSlot;
                const int nk = warp < nblk ? (nblk - 1 - warp) / kWarps + 1 : 0;
                const int hd = dd >> 1;  // 16-byte chunks per encW row (<= 8)
                const int er0 = lane >> 3, ec = lane & 7;
                auto stage = [&](int k) {
                    if (k < nk) {
                        const int b = warp + k * kWarps;
                        double *sl = ring + (k & 3) * kDmsSlot;
                        const double *gp = proj + (size_t)(8 * b) * kH + 2 * lane;
#pragma unroll
                        for (int r = 0; r < 8; r++)
                            cp_async16(sl + dms_p(r, 2 * lane), gp + (8 * b + r < T ? r * kH : 0), 8 * b + r < T);
#pragma unroll
                        for (int h2 = 0; h2 < 2; h2++) {
                            const int r = er0 + 4 * h2, row = 8 * b + r;
                            if (ec < hd)
                                cp_async16(sl + dms_e(r, 2 * ec), encW + (size_t)(row < T ? row : 0) * dd + 2 * ec,
                                           row < T);
                        }
                    }
                    cp_async_commit();
                };
                stage(0);
                stage(1);
                double ua[2][2][2] = {};  // [block parity][n][e]: uc[sample fg][8 n + 2 ft + e]
                double es = 0.0;          // sum of e[sample fg] over this lane's rows
                for (int k = 0; k < nk; k += 2) {
                    stage(k + 2);
                    stage(k + 3);
                    cp_async_wait<2>();
                    __syncwarp();
                    double a4[2][4][2];
#pragma unroll
                    for (int bb = 0; bb < 2; bb++)
#pragma unroll
                        for (int q = 0; q < 4; q++) a4[bb][q][0] = a4[bb][q][1] = 0.0;
#pragma unroll
                    for (int ks = 0; ks < kH / 4; ks++)
#pragma unroll
                        for (int bb = 0; bb < 2; bb++)
                            dmma_f64(a4[bb][ks & 3], bf[ks], ring[((k + bb) & 3) * kDmsSlot + dms_p(fg, 4 * ks + ft)]);
#pragma unroll
                    for (int bb = 0; bb < 2; bb++) {
                        const int b = warp + (k + bb) * kWarps;
                        const double *se = ring + ((k + bb) & 3) * kDmsSlot;
                        double ev[2];
#pragma unroll
                        for (int e = 0; e < 2; e++) {
                            const int i = 8 * b + 2 * ft + e;
                            const double sv = (a4[bb][0][e] + a4[bb][1][e]) + (a4[bb][2][e] + a4[bb][3][e]);
                            ev[e] = (k + bb < nk && i < T) ? fm_exp(sv) : 0.0;
                            es += ev[e];
                            if (a.act_e && k + bb < nk && i < T && fg < Mb)
                                a.act_e[((size_t)(k0 + fg) * T + t) * T + i] = ev[e];
                        }
#pragma unroll
                        for (int e = 0; e < 2; e++)
#pragma unroll
                            for (int n = 0; n < 2; n++)
                                if (n * 8 < dd) dmma_f64(ua[bb][n], ev[e], se[dms_e(2 * ft + e, 8 * n + fg)]);
                    }
                    __syncwarp();  // slots (k, k + 1) & 3 are restaged next iteration
                }
                cp_async_wait<0>();
                es += __shfl_xor_sync(0xffffffffu, es, 1);
                es += __shfl_xor_sync(0xffffffffu, es, 2);
#pragma unroll
                for (int m = 0; m < MT; m++) lsm[m] = __shfl_sync(0xffffffffu, es, 4 * m);
#pragma unroll
                for (int n = 0; n < 2; n++)
#pragma unroll
                    for (int e = 0; e < 2; e++) {
                        const int j = 8 * n + 2 * ft + e;
                        if (j < dd && fg < Mb) puc[(warp * M + fg) * dd + j] = ua[0][n][e] + ua[1][n][e];
                    }
            }
#pragma unroll 2
            for (int blk = warp; blk < (dms ? 0 : nblk); blk += kWarps) {
                const int i = blk * 8 + fg;
                const double *pr = proj + (size_t)(i < T ? i : T - 1) * kH + ft;
                double acc[2] = {0.0, 0.0};
#pragma unroll
                for (int ks = 0; ks < kH / 4; ks++) dmma_f64(acc, __ldg(pr + 4 * ks), bf[ks]);
                if (i < T) {
                    alS[(2 * ft) * a.Tpad + i] = acc[0];      // sample 2t
                    alS[(2 * ft + 1) * a.Tpad + i] = acc[1];  // sample 2t + 1
                }
            }
            if (!dms) __syncthreads();  // the exp loop reads rows other warps scored
            if (!noshift)
                for (int i = tid; i < T; i += kThreads)
#pragma unroll
                    for (int m = 0; m < MT; m++) lmx[m] = fmax(lmx[m], alS[m * a.Tpad + i]);
        } else if (TCG) {
            // scores only: this thread's proj row is in registers (w), h is broadcast
            // from shared memory; the next step's h W_h is on the tensor cores
            double s0[MT], s1[MT], s2[MT], s3[MT];
#pragma unroll
            for (int m = 0; m < MT; m++) s0[m] = s1[m] = s2[m] = s3[m] = 0.0;
#pragma unroll
            for (int j2 = 0; j2 < kH / 2; j2 += 2) {
#pragma unroll
                for (int m = 0; m < MT; m++) {
                    const double2 h0 = reinterpret_cast<const double2 *>(hcur[m])[j2];
                    const double2 h1 = reinterpret_cast<const double2 *>(hcur[m])[j2 + 1];
                    s0[m] = fma(w[2 * j2], h0.x, s0[m]);
                    s1[m] = fma(w[2 * j2 + 1], h0.y, s1[m]);
                    s2[m] = fma(w[2 * j2 + 2], h1.x, s2[m]);
                    s3[m] = fma(w[2 * j2 + 3], h1.y, s3[m]);
                }
            }
#pragma unroll
            for (int m = 0; m < MT; m++)
                if (m < Mb && tid < T) {
                    const double sv = (s0[m] + s1[m]) + (s2[m] + s3[m]);
                    if (!FAST) alS[m * a.Tpad + tid] = sv;
                    sreg[m] = sv;
                    lmx[m] = sv;
                }
        } else {
            // fused pass: this thread's first score row and its gate column of the
            // next step's h W_h share every h load (W_h indices stay compile-time)
            const int i = tid < T ? tid : T - 1;
            const double2 *pr = reinterpret_cast<const double2 *>(proj + (size_t)i * LD);
            // 4 independent accumulators per dot (short FMA dependency chains)
            double s0[MT], s1[MT], s2[MT], s3[MT], g0[MT], g1[MT], g2[MT], g3[MT];
#pragma unroll
            for (int m = 0; m < MT; m++) s0[m] = s1[m] = s2[m] = s3[m] = g0[m] = g1[m] = g2[m] = g3[m] = 0.0;
#pragma unroll
            for (int j2 = 0; j2 < kH / 2; j2 += 2) {
                const double2 e0 = pr[j2], e1 = pr[j2 + 1];
#pragma unroll
                for (int m = 0; m < MT; m++) {
                    const double2 h0 = reinterpret_cast<const double2 *>(hcur[m])[j2];
                    const double2 h1 = reinterpret_cast<const double2 *>(hcur[m])[j2 + 1];
                    s0[m] = fma(e0.x, h0.x, s0[m]);
                    s1[m] = fma(e0.y, h0.y, s1[m]);
                    s2[m] = fma(e1.x, h1.x, s2[m]);
                    s3[m] = fma(e1.y, h1.y, s3[m]);
                    g0[m] = fma(h0.x, w[2 * j2], g0[m]);
                    g1[m] = fma(h0.y, w[2 * j2 + 1], g1[m]);
                    g2[m] = fma(h1.x, w[2 * j2 + 2], g2[m]);
                    g3[m] = fma(h1.y, w[2 * j2 + 3], g3[m]);
                }
            }
#pragma unroll
            for (int m = 0; m < MT; m++)
                if (m < Mb) {
                    gn[m] = (g0[m] + g1[m]) + (g2[m] + g3[m]);
                    if (SPEC) gnS[m * kG + col] = gn[m];
                    if (tid < T) {
                        const double s = (s0[m] + s1[m]) + (s2[m] + s3[m]);
                        if (!FAST) alS[m * a.Tpad + tid] = s;
                        sreg[m] = s;
                        lmx[m] = s;
                    }
                }
        }
        for (int i = tid + kThreads; i < ((FAST || DM) ? 0 : T); i += kThreads) {
            const double2 *pr = reinterpret_cast<const double2 *>(proj + (size_t)i * LD);
            double s0[MT], s1[MT];
#pragma unroll
            for (int m = 0; m < MT; m++) s0[m] = s1[m] = 0.0;
#pragma unroll 8
            for (int j2 = 0; j2 < kH / 2; j2++) {
                const double2 e = pr[j2];
#pragma unroll
                for (int m = 0; m < MT; m++) {
                    const double2 hh = reinterpret_cast<const double2 *>(hcur[m])[j2];
                    s0[m] = fma(e.x, hh.x, s0[m]);
                    s1[m] = fma(e.y, hh.y, s1[m]);
                }
            }
#pragma unroll
            for (int m = 0; m < MT; m++)
                if (m < Mb) {
                    const double s = s0[m] + s1[m];
                    alS[m * a.Tpad + i] = s;
                    lmx[m] = fmax(lmx[m], s);
                }
        }
#pragma unroll
        for (int m = 0; m < MT; m++) lmx[m] = noshift ? 0.0 : warp_max(lmx[m]);
        for (int i = tid; i < ((skip & 16) || dms ? 0 : T); i += kThreads) {
            double ev[MT];
#pragma unroll
            for (int m = 0; m < MT; m++) ev[m] = fm_exp((FAST ? sreg[m] : alS[m * a.Tpad + i]) - lmx[m]);
#pragma unroll
            for (int m = 0; m < MT; m++)
                if (m < Mb) {
                    alS[m * a.Tpad + i] = ev[m];
                    lsm[m] += ev[m];
                    if (a.act_e) a.act_e[((size_t)(k0 + m) * T + t) * T + i] = ev[m];
                }
        }
#pragma unroll
        for (int m = 0; m < MT; m++)
            lsm[m] = ((skip & 8) || (FAST && (MT == 2 || MT == 4)) || dms) ? lsm[m] : warp_sum(lsm[m]);
        __syncwarp();
        // uc_w[m][j] = sum over this warp's rows {32 warp + 256 r + l} of e_i encW[i][j]
        // (lane = (m, j); full 32-row blocks read e and encW^T as 16-byte pairs)
        double ucv = 0.0;  // this lane's uc_w[m][j] (first pass)
        if (DM) {
            // fp64 tensor-core tiles: uc_w[m][j] = sum over the warp's rows of e[m][i]
            // encW[i][j] (m = the 8 samples, j in 8-column tiles, k = rows)
            const int fg = lane >> 2, ft = lane & 3;
            constexpr int kNtMax = kMaxDD / 8;
            const int ntl = (dd + 7) >> 3;
            double acc[kNtMax][2];
#pragma unroll
            for (int n = 0; n < kNtMax; n++) acc[n][0] = acc[n][1] = 0.0;
            for (int ib = warp * 32; ib < ((skip & 1) || dms ? 0 : T); ib += kThreads) {
#pragma unroll
                for (int ks = 0; ks < 8; ks++) {
                    const int i = ib + 4 * ks + ft;
                    const bool ok = i < T;
                    const double ae = ok ? alS[fg * a.Tpad + i] : 0.0;  // A[m = g][k = t]
                    const double *ew = encW + (size_t)(ok ? i : 0) * dd;
#pragma unroll
                    for (int n = 0; n < kNtMax; n++)
                        if (n < ntl) {
                            const int j = 8 * n + fg;
                            dmma_f64(acc[n], ae, j < dd ? __ldg(ew + j) : 0.0);  // B[k = t][n = g]
                        }
                }
            }
#pragma unroll
            for (int n = 0; n < kNtMax; n++)
#pragma unroll
                for (int e = 0; e < 2; e++) {
                    const int j = 8 * n + 2 * ft + e;
                    if (n < ntl && j < dd && fg < Mb && !dms) puc[(warp * M + fg) * dd + j] = acc[n][e];
                }
        } else if (FAST && MT == 2) {
            // lane (j, half): 16 of the warp's 32 rows for both samples, so each
            // encW^T pair is loaded once for the two samples; halves combine
            // with one shuffle (2/3 of the generic loop's shared-memory wavefronts)
            const int j = lane & 15, hh = lane >> 4, jj = j < dd ? j : dd - 1;
            const int i0 = warp * 32 + hh * 16, n = (skip & 1) ? 0 : max(0, min(16, T - i0));
            // the same pass also sums the e values (the warp's softmax partial sum,
            // in place of a 5-level butterfly): every lane of a half holds it
            double c0 = 0.0, c1 = 0.0, d0 = 0.0, d1 = 0.0, s0 = 0.0, s1 = 0.0;
            if (n == 16) {
                const double2 *ap0 = reinterpret_cast<const double2 *>(alS + i0);
                const double2 *ap1 = reinterpret_cast<const double2 *>(alS + a.Tpad + i0);
                const double2 *ep = reinterpret_cast<const double2 *>(encW + jj * a.ewld + i0);
#pragma unroll
                for (int q = 0; q < 8; q++) {
                    const double2 e = ep[q], x = ap0[q], y = ap1[q];
                    c0 = fma(x.x, e.x, c0);
                    c1 = fma(x.y, e.y, c1);
                    d0 = fma(y.x, e.x, d0);
                    d1 = fma(y.y, e.y, d1);
                    s0 += x.x + x.y;
                    s1 += y.x + y.y;
                }
            } else {
                for (int ii = 0; ii < n; ii++) {
                    const double e = encW[jj * a.ewld + i0 + ii];
                    c0 = fma(alS[i0 + ii], e, c0);
                    d0 = fma(alS[a.Tpad + i0 + ii], e, d0);
                    s0 += alS[i0 + ii];
                    s1 += alS[a.Tpad + i0 + ii];
                }
            }
            double v0 = c0 + c1, v1 = d0 + d1;
            v0 += __shfl_xor_sync(0xffffffffu, v0, 16);
            v1 += __shfl_xor_sync(0xffffffffu, v1, 16);
            s0 += __shfl_xor_sync(0xffffffffu, s0, 16);
            s1 += __shfl_xor_sync(0xffffffffu, s1, 16);
            if (!(skip & 8)) {
                lsm[0] = s0;
                lsm[1] = s1;
            }
            if (j < dd) puc[(warp * M + hh) * dd + j] = hh ? v1 : v0;
        } else if (FAST && MT == 4) {
            // lane (j, pair): all 32 of the warp's rows for samples 2 pair and 2 pair + 1, each
            // encW^T pair loaded once for two samples; the same pass sums the e values (the
            // warp's softmax partial sums, no butterflies)
            const int j = lane & 15, pr = lane >> 4, jj = j < dd ? j : dd - 1;
            const int i0 = warp * 32, n = (skip & 1) ? 0 : max(0, min(32, T - i0));
            double c0 = 0.0, c1 = 0.0, d0 = 0.0, d1 = 0.0, s0 = 0.0, s1 = 0.0;
            const double *a0p = alS + (2 * pr) * a.Tpad + i0, *a1p = a0p + a.Tpad;
            if (n == 32) {
                const double2 *ap0 = reinterpret_cast<const double2 *>(a0p);
                const double2 *ap1 = reinterpret_cast<const double2 *>(a1p);
                const double2 *ep = reinterpret_cast<const double2 *>(encW + jj * a.ewld + i0);
#pragma unroll
                for (int q = 0; q < 16; q++) {
                    const double2 e = ep[q], x = ap0[q], y = ap1[q];
                    c0 = fma(x.x, e.x, c0);
                    c1 = fma(x.y, e.y, c1);
                    d0 = fma(y.x, e.x, d0);
                    d1 = fma(y.y, e.y, d1);
                    s0 += x.x + x.y;
                    s1 += y.x + y.y;
                }
            } else {
                for (int ii = 0; ii < n; ii++) {
                    const double e = encW[jj * a.ewld + i0 + ii];
                    c0 = fma(a0p[ii], e, c0);
                    d0 = fma(a1p[ii], e, d0);
                    s0 += a0p[ii];
                    s1 += a1p[ii];
                }
            }
            if (!(skip & 8)) {
                lsm[0] = __shfl_sync(0xffffffffu, s0, 0);
                lsm[1] = __shfl_sync(0xffffffffu, s1, 0);
                lsm[2 % MT] = __shfl_sync(0xffffffffu, s0, 16);
                lsm[3 % MT] = __shfl_sync(0xffffffffu, s1, 16);
            }
            if (j < dd) {
                if (2 * pr < Mb) puc[(warp * M + 2 * pr) * dd + j] = c0 + c1;
                if (2 * pr + 1 < Mb) puc[(warp * M + 2 * pr + 1) * dd + j] = d0 + d1;
            }
        } else
        for (int pi = lane; pi < ((skip & 1) ? 0 : Mb * dd); pi += 32) {
            const int m = small_div<MT>(pi, dd), j = pi - m * dd;
            const double *al = alS + m * a.Tpad;
            double c0 = 0.0, c1 = 0.0, c2 = 0.0, c3 = 0.0;
            for (int i0 = warp * 32; i0 < T; i0 += kThreads) {
                const int n = min(32, T - i0);
                if (PS && n == 32) {
                    const double2 *ap = reinterpret_cast<const double2 *>(al + i0);
                    const double2 *ep = reinterpret_cast<const double2 *>(encW + j * a.ewld + i0);
#pragma unroll
                    for (int q = 0; q < 16; q += 2) {
                        const double2 a0 = ap[q], a1 = ap[q + 1], e0 = ep[q], e1 = ep[q + 1];
                        c0 = fma(a0.x, e0.x, c0);
                        c1 = fma(a0.y, e0.y, c1);
                        c2 = fma(a1.x, e1.x, c2);
                        c3 = fma(a1.y, e1.y, c3);
                    }
                } else {
                    for (int ii = 0; ii < n; ii++) {
                        const int i = i0 + ii;
                        const double ew = PS ? encW[j * a.ewld + i] : encW[(size_t)i * dd + j];
                        c0 = fma(al[i], ew, c0);
                    }
                }
            }
            const double v = (c0 + c1) + (c2 + c3);
            puc[(warp * M + m) * dd + j] = v;
            if (pi == lane) ucv = v;
        }
        if (lane == 0) {
#pragma unroll
            for (int m = 0; m < MT; m++)
                if (m < Mb) {
                    pmx[warp * M + m] = lmx[m];
                    psm[warp * M + m] = lsm[m];
                }
        }
        // fast E (D <= 4, dd <= 16, spare warps): the draw warp forms the logits
        // itself (h . vdev + dev_table . sum_w uc_w) -> no pz partials, no uh here
        const bool fastE = FAST || (D <= 4 && dd <= 16 && 2 * Mb <= kWarps);
        // pz_w[m][d] = dev_table[d] . uc_w[m]
        if (fastE) {
        } else if (dd == 16 && Mb <= 2) {
            // lanes (m, j) hold uc_w[m][j]: per device, a 16-lane butterfly sum
            const int m = lane >> 4, j = lane & 15;
            for (int d0 = 0; d0 < ((skip & 2) ? 0 : D); d0 += 4) {
                double v[4];
#pragma unroll
                for (int q = 0; q < 4; q++) v[q] = d0 + q < D ? devt[(d0 + q) * 16 + j] * ucv : 0.0;
#pragma unroll
                for (int o = 8; o > 0; o >>= 1)
#pragma unroll
                    for (int q = 0; q < 4; q++) v[q] += __shfl_xor_sync(0xffffffffu, v[q], o);
                if (j == 0 && m < Mb)
#pragma unroll
                    for (int q = 0; q < 4; q++)
                        if (d0 + q < D) pz[(warp * M + m) * D + d0 + q] = v[q];
            }
        } else {
        __syncwarp();
        for (int pi = lane; pi < ((skip & 2) ? 0 : Mb * D); pi += 32) {
            const int m = small_div<MT>(pi, D), d = pi - m * D;
            const double *pv = puc + (warp * M + m) * dd;
            double z0 = 0.0, z1 = 0.0;
            int o = 0;
            for (; o + 2 <= dd; o += 2) {
                z0 = fma(devt[d * dd + o], pv[o], z0);
                z1 = fma(devt[d * dd + o + 1], pv[o + 1], z1);
            }
            if (o < dd) z0 = fma(devt[d * dd + o], pv[o], z0);
            pz[(warp * M + m) * D + d] = z0 + z1;
        }
        }
        // uh = h @ W_out[:64] (policy.py:302, h half), 8 lanes per output
        // (fast E: the spare warps form it during E, off the draw chain)
        if (!fastE) {
            const int total = (skip & 4) ? 0 : Mb * dd * 8;
            for (int b0 = 0; b0 < total; b0 += kThreads) {
                const int idx = b0 + tid;
                const bool ok = idx < total;
                double part = 0.0;
                int m = 0, o = 0;
                if (ok) {
                    const int pair = idx >> 3, pp = idx & 7;
                    m = small_div<MT>(pair, dd);
                    o = pair - m * dd;
                    const double *hv = (SPEC ? hC + (m * D + prv[m]) * kH : hS + m * kH) + pp;
                    const double *wc = wout1 + o * kWout1Ld + pp;
                    double p0 = 0.0, p1 = 0.0;
#pragma unroll
                    for (int y = 0; y < 8; y += 2) {
                        p0 = fma(hv[8 * y], wc[8 * y], p0);
                        p1 = fma(hv[8 * y + 8], wc[8 * y + 8], p1);
                    }
                    part = p0 + p1;
                }
                part += __shfl_xor_sync(0xffffffffu, part, 4);
                part += __shfl_xor_sync(0xffffffffu, part, 2);
                part += __shfl_xor_sync(0xffffffffu, part, 1);
                if (ok && (idx & 7) == 0) uhS[m * 32 + o] = part;
            }
        }
        DP_WEND(1);
        __syncthreads();
        DP_WSTART();
        DP_PHASE(1);
        // ---- E: combine, logits, softmax over devices, draw (policy.py:297-308, 320-323) ----
        // warp m < Mb runs sample m's draw chain; when there are spare warps, warp
        // Mb + m does the sample's off-chain stores (u, uc, the alpha scales)
        const bool split = FAST || 2 * Mb <= kWarps;
        // the draw warps' chain first in program order: they fall through into it
        // after the barrier (the helper / pcg warps jump)
        for (int m = warp; m < Mb; m += kWarps) {
            const size_t row = (size_t)(k0 + m) * T + t;
            // the step's uniform: precomputed by the pcg warp, or (no spare warps)
            // stepped here — every lane steps the same PCG64 state, lane 0 keeps it
            u128 rs{0, 0};
            double r;
            if (pcgw) {
                r = rnext[par * M + m];
            } else {
                rs = pcg_step(u128{pcg[2 * m], pcg[2 * m + 1]}, u128{a.inc_hi, a.inc_lo});
                r = pcg_double(rs);
            }
            double gmx = 0.0, f = lane < kWarps ? 1.0 : 0.0;
            double fw[kWarps];
#pragma unroll
            for (int ww = 0; ww < kWarps; ww++) fw[ww] = 1.0;
            if (!noshift) {
                gmx = pmx[m];
#pragma unroll
                for (int ww = 1; ww < kWarps; ww++) gmx = fmax(gmx, pmx[ww * M + m]);
                f = lane < kWarps ? fm_exp(pmx[(lane & (kWarps - 1)) * M + m] - gmx) : 0.0;
#pragma unroll
                for (int ww = 0; ww < kWarps; ww++) fw[ww] = __shfl_sync(0xffffffffu, f, ww);
            }
            // sum of the 8 warp partials as a 3-level tree (chain depth 4, not 8)
            const double gsum = wsum8(psm + m, M, fw);
            if (!split && a.act_esc && lane < kWarps) a.act_esc[row * kWarps + lane] = fm_div(f, gsum);
            // all lanes compute (clamped indices, no divergent branches: the z, uc
            // and pcg chains interleave); lanes >= D / >= dd are masked at the end
            const int ld = lane < D ? lane : D - 1, lo = lane < dd ? lane : dd - 1;
            double zh, zcd = 0.0;
            if (fastE) {
                // lanes (d = lane / 8, part = lane % 8): h . vdev[:, d] (8 terms each)
                // and dev_table[d] . sum_w uc_w (2 terms each), 3-level butterflies
                // (D <= 8: lanes (d = lane / 4, part = lane % 4), 16 + 4 terms, 2 levels)
                const int dz = min(lane / NP, D - 1), op = lane % NP;
                const double *hv = SPEC ? hC + (m * D + prv[m]) * kH : hS + m * kH;
                double v0 = 0.0, v1 = 0.0;
#pragma unroll
                for (int y = 0; y < kH / NP; y += 2) {
                    v0 = fma(hv[op + NP * y], vS[(op + NP * y) * D + dz], v0);
                    v1 = fma(hv[op + NP * y + NP], vS[(op + NP * y + NP) * D + dz], v1);
                }
                // 1 / gsum off the chain (the loads above are in flight); the context
                // half joins the h half before one butterfly
                const double rg = fm_div(1.0, gsum);
                const double ucr = wsum8(puc + m * dd + lo, M * dd, fw);  // lane j < dd: sum_w fw[w] uc_w[j]
                const double ua = __shfl_sync(0xffffffffu, ucr, op), ub = __shfl_sync(0xffffffffu, ucr, op + NP);
                double c = op < dd ? devt[dz * dd + op] * ua : 0.0;
                if (op + NP < dd) c = fma(devt[dz * dd + op + NP], ub, c);
#pragma unroll
                for (int q = 2; q < 16 / NP; q++) {
                    const int j = op + NP * q;
                    const double uq = __shfl_sync(0xffffffffu, ucr, j);
                    if (j < dd) c = fma(devt[dz * dd + j], uq, c);
                }
                double v = fma(c, rg, v0 + v1);
#pragma unroll
                for (int o = 1; o < NP; o <<= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
                zh = __shfl_sync(0xffffffffu, v, ld * NP);
            } else if (D <= 4 && dd <= 16) {
                // lanes (d = lane / 8, part = lane % 8): 2 terms each + a 3-level butterfly
                const int dz = min(lane >> 3, D - 1), op = lane & 7;
                double v = op < dd ? devt[dz * dd + op] * uhS[m * 32 + op] : 0.0;
                if (op + 8 < dd) v = fma(devt[dz * dd + op + 8], uhS[m * 32 + op + 8], v);
                v += __shfl_xor_sync(0xffffffffu, v, 1);
                v += __shfl_xor_sync(0xffffffffu, v, 2);
                v += __shfl_xor_sync(0xffffffffu, v, 4);
                zh = __shfl_sync(0xffffffffu, v, ld * 8);
            } else {
                double zh0 = 0.0, zh1 = 0.0;
                int o = 0;
                for (; o + 2 <= dd; o += 2) {
                    zh0 = fma(devt[ld * dd + o], uhS[m * 32 + o], zh0);
                    zh1 = fma(devt[ld * dd + o + 1], uhS[m * 32 + o + 1], zh1);
                }
                if (o < dd) zh0 = fma(devt[ld * dd + o], uhS[m * 32 + o], zh0);
                zh = zh0 + zh1;
            }
            double zv;
            if (fastE) {
                zv = zh + bout[ld];  // zh carries the context half
            } else {
                double zc = zcd;
#pragma unroll
                for (int ww = 0; ww < kWarps; ww++) zc = fma(pz[(ww * M + m) * D + ld], fw[ww], zc);
                zv = (zh + fm_div(zc, gsum)) + bout[ld];
            }
            const double z = lane < D ? zv : -INFINITY;
            if (!split) {
                // u (and its context half uc) for the backward
                double uc = 0.0;
#pragma unroll
                for (int ww = 0; ww < kWarps; ww++) uc = fma(puc[(ww * M + m) * dd + lo], fw[ww], uc);
                const double ucn = fm_div(uc, gsum);
                if (lane < dd) {
                    a.act_u[row * dd + lane] = uhS[m * 32 + lane] + ucn;
                    a.act_uc[row * dd + lane] = ucn;
                }
            }
            double zmax = z;
#pragma unroll
            for (int o = FAST ? DX / 2 : 16; o > 0; o >>= 1) {  // FAST: D <= DX, lanes >= D hold -inf
                const double oz = __shfl_xor_sync(0xffffffffu, zmax, o);
                // FAST: compare-select (~12 cycles) in place of fmax (~25); z is finite
                if (FAST) zmax = oz > zmax ? oz : zmax;
                else if (o < d_pow2) zmax = fmax(zmax, oz);
            }
            const double zs = z - zmax;
            const double ezv = fm_exp(lane < D ? zs : -1000.0);
            const double ez = lane < D ? ezv : 0.0;
            if (FAST) {
                // the draw itself, nothing else on the chain: the cumulative sums of the
                // 4 exponentials in numpy's order (cumsum / pairwise_sum with n < 8 are
                // sequential; lanes >= D add exact zeros, so P[3] == esum) against r * esum
                // — searchsorted(cumsum(ez / esum), r, 'right') without the division.
                // p = ez / esum, the margin and the row's global stores are the pcg
                // warp's, one step later (fin_store).  The decision agrees with the
                // reference's whenever the margin recorded there exceeds
                // SAMPLING_MARGIN_TOL (cumsum(p) and P / esum differ by a few ulp).
                double P[DX];
                P[0] = __shfl_sync(0xffffffffu, ez, 0);
#pragma unroll
                for (int dv = 1; dv < DX; dv++) P[dv] = P[dv - 1] + __shfl_sync(0xffffffffu, ez, dv);
                const double esum = P[DX - 1];
                int ch;
                if (a.forced) {
                    ch = a.forced[row];
                } else {
                    const double rs = r * esum;
                    int cnt = 0;
#pragma unroll
                    for (int dv = 0; dv < DX - 1; dv++) cnt += (dv < D - 1 && P[dv] <= rs) ? 1 : 0;
                    ch = cnt;
                }
                double *f = fin + (par * M + m) * FS;
                if (lane == 0) prev[(par ^ 1) * M + m] = ch;
                if (lane < D) {
                    f[4 + lane] = zs;
                    f[EZO + lane] = ez;
                }
                if (lane == 0) {
                    f[0] = esum;
                    f[1] = gmx;
                    f[2] = gsum;
                }
                continue;
            }
            // numpy pairwise order over the D terms (np_sum_small), identical in every lane
            double esum;
            if (D < 8) {
                double ev[8];
#pragma unroll
                for (int dv = 0; dv < 8; dv++) ev[dv] = __shfl_sync(0xffffffffu, ez, dv);
                esum = 0.0;
#pragma unroll
                for (int dv = 0; dv < 8; dv++)
                    if (dv < D) esum += ev[dv];
            } else {
                double rr[8];
#pragma unroll
                for (int j = 0; j < 8; j++) rr[j] = __shfl_sync(0xffffffffu, ez, j);
                int i = 8;
                for (; i < D - (D % 8); i += 8) {
#pragma unroll
                    for (int j = 0; j < 8; j++) rr[j] += __shfl_sync(0xffffffffu, ez, i + j);
                }
                esum = ((rr[0] + rr[1]) + (rr[2] + rr[3])) + ((rr[4] + rr[5]) + (rr[6] + rr[7]));
                for (; i < D; i++) esum += __shfl_sync(0xffffffffu, ez, i);
            }
            const double pr = fm_div(ez, esum);
            if (lane < D) {
                a.act_p[row * D + lane] = pr;
                if (a.probs_out) a.probs_out[row * D + lane] = pr;
            }
            int ch;
            if (a.forced) {
                ch = a.forced[row];
            } else {
                double cdf = 0.0, mg = INFINITY;
                int cnt = 0;
                // margin: distance of the uniform to every cdf boundary that can
                // change the choice (j < D-1; the last one is clamped away)
                const bool wm = a.margin != nullptr;
                if (D <= 8) {
                    double pv[8];
#pragma unroll
                    for (int dv = 0; dv < 8; dv++) pv[dv] = __shfl_sync(0xffffffffu, pr, dv);
#pragma unroll
                    for (int dv = 0; dv < 8; dv++)
                        if (dv < D) {
                            cdf += pv[dv];
                            cnt += (cdf <= r) ? 1 : 0;
                            if (wm && dv < D - 1) mg = fmin(mg, fabs(r - cdf));
                        }
                } else {
                    for (int dv = 0; dv < D; dv++) {
                        cdf += __shfl_sync(0xffffffffu, pr, dv);
                        cnt += (cdf <= r) ? 1 : 0;
                        if (wm && dv < D - 1) mg = fmin(mg, fabs(r - cdf));
                    }
                }
                mrun = fmin(mrun, mg);
                ch = cnt < D - 1 ? cnt : D - 1;
            }
            const double zsc = __shfl_sync(0xffffffffu, zs, ch);
            if (!a.forced && !pcgw) __syncwarp();  // every lane's read of pcg[] precedes lane 0's write
            if (lane == 0) {
                if (!a.forced && !pcgw) {
                    pcg[2 * m] = rs.hi;
                    pcg[2 * m + 1] = rs.lo;
                }
                prev[(par ^ 1) * M + m] = ch;
                a.choice[row] = (uint8_t)ch;
                if (a.choice_out) a.choice_out[row] = (uint8_t)ch;
                a.act_lz[row * 2] = zsc;
                a.act_lz[row * 2 + 1] = esum;
                // softmax stats (max, sum) for the backward's recompute of alpha
                a.act_stat[row * 2] = gmx;
                a.act_stat[row * 2 + 1] = gsum;
            }
        }
        if (split && warp >= Mb && warp < 2 * Mb) {
            const int m = warp - Mb;
            const size_t row = (size_t)(k0 + m) * T + t;
            double gmx = 0.0, f = lane < kWarps ? 1.0 : 0.0;
            double fw[kWarps];
#pragma unroll
            for (int ww = 0; ww < kWarps; ww++) fw[ww] = 1.0;
            if (!noshift) {
                gmx = pmx[m];
#pragma unroll
                for (int ww = 1; ww < kWarps; ww++) gmx = fmax(gmx, pmx[ww * M + m]);
                f = lane < kWarps ? fm_exp(pmx[(lane & (kWarps - 1)) * M + m] - gmx) : 0.0;
#pragma unroll
                for (int ww = 0; ww < kWarps; ww++) fw[ww] = __shfl_sync(0xffffffffu, f, ww);
            }
            double gsum = 0.0;
#pragma unroll
            for (int ww = 0; ww < kWarps; ww++) gsum = fma(psm[ww * M + m], fw[ww], gsum);
            if (a.act_esc && lane < kWarps) a.act_esc[row * kWarps + lane] = fm_div(f, gsum);
            const int lo = lane < dd ? lane : dd - 1;
            double uc = 0.0;
#pragma unroll
            for (int ww = 0; ww < kWarps; ww++) uc = fma(puc[(ww * M + m) * dd + lo], fw[ww], uc);
            const double ucn = fm_div(uc, gsum);
            double uh;
            if (fastE) {
                // uh[o] = h . W_out[:64, o]: lanes (o, half) sum 32 terms each
                const double *hv = (SPEC ? hC + (m * D + prv[m]) * kH : hS + m * kH) + (lane >> 4) * 32;
                const double *wc = woS + (lane >> 4) * 32 * dd + ((lane & 15) < dd ? (lane & 15) : dd - 1);
                double u0 = 0.0, u1 = 0.0, u2 = 0.0, u3 = 0.0;
#pragma unroll
                for (int l = 0; l < 32; l += 4) {
                    u0 = fma(hv[l], wc[l * dd], u0);
                    u1 = fma(hv[l + 1], wc[(l + 1) * dd], u1);
                    u2 = fma(hv[l + 2], wc[(l + 2) * dd], u2);
                    u3 = fma(hv[l + 3], wc[(l + 3) * dd], u3);
                }
                const double part = (u0 + u1) + (u2 + u3);
                uh = part + __shfl_xor_sync(0xffffffffu, part, 16);
            } else {
                uh = uhS[m * 32 + lo];
            }
            if (lane < dd) {
                a.act_u[row * dd + lane] = uh + ucn;
                a.act_uc[row * dd + lane] = ucn;
            }
        }
        // pcg warps: the last Mb warps — on the sub-partitions of the split warps
        // (warp w issues on SMSP w % 4), not sharing issue slots with the draw warps
        if (pcgw && warp >= kWarps - Mb && lane == 0) {
            const int m = warp - (kWarps - Mb);
            // the previous step's row (reads that step's uniform before it is overwritten)
            if (FAST && t > 0) fin_store<FS, EZO>(a, fin, prev, rnext, k0, m, M, T, t - 1);
            if (!a.forced) {
                const u128 ns = pcg_step(u128{pcg[2 * m], pcg[2 * m + 1]}, u128{a.inc_hi, a.inc_lo});
                pcg[2 * m] = ns.hi;
                pcg[2 * m + 1] = ns.lo;
                rnext[(par ^ 1) * M + m] = pcg_double(ns);
            }
        }
        if (SPEC && warp >= Mb && t + 1 < T) {
            // next step's LSTM cell for every possible choice d (the idle warps)
            const int st = tid - Mb * 32, nst = kThreads - Mb * 32;
            const int n_items = Mb * D * kH;
#pragma unroll 2
            for (int it = st; it < n_items; it += nst) {
                const int m = it / (D * kH), rem = it - m * D * kH, d = rem >> 6, uu = rem & 63;
                const double *g = gnS + m * kG + uu;
                const double *ed = edev + d * kG + uu;
                const double ai = gate_act(__ldg(ed) + g[0], false);
                const double af = gate_act(__ldg(ed + kH) + g[kH], false);
                const double ao = gate_act(__ldg(ed + 2 * kH) + g[2 * kH], false);
                const double ag = gate_act(__ldg(ed + 3 * kH) + g[3 * kH], true);
                const double cold = cC[(par * M * D + m * D + prv[m]) * kH + uu];
                const double cn = af * cold + ai * ag;
                const double hn = ao * tanh_x(cn);
                double *ac = aC + (m * D + d) * kG + uu;
                ac[0] = ai;
                ac[kH] = af;
                ac[2 * kH] = ao;
                ac[3 * kH] = ag;
                hC[(m * D + d) * kH + uu] = hn;
                cC[((par ^ 1) * M * D + m * D + d) * kH + uu] = cn;
            }
        }
        if (!SPEC) {
            // gn for the non-speculative A of the next step is already in registers
        }
        DP_WEND(2);
        __syncthreads();
        DP_WSTART();
        DP_PHASE(2);
    }
#undef DP_PHASE
#undef DP_WEND
#undef DP_WSTART
    if (wclk)
#pragma unroll
        for (int i = 0; i < 3; i++) g_warp_clk[warp * 3 + i] += wacc[i];
    if (FAST && tid < Mb && T > 0) {
        fin_store<FS, EZO>(a, fin, prev, rnext, k0, tid, M, T, T - 1);  // the last step's row
        if (a.margin && !a.forced) a.margin[k0 + tid] = fin[2 * FS * M + tid];
    }
    if (!FAST && a.margin && !a.forced && warp < Mb && lane == 0) a.margin[k0 + warp] = mrun;
    __syncthreads();  // the log-prob pass below reads those rows from other threads
    if (TCG && warp == 0) {
        tc::fence_after();
        tc::tmem_dealloc(tm, kTmCols);
    }
    if (clk_on)
#pragma unroll
        for (int i = 0; i < 3; i++) g_phase_clk[i] += clk_acc[i];
    // ---- log p = sum_t (zs[c_t] - log sum_t): logs in parallel, sum in t order ----
    __threadfence_block();
    for (int m = 0; m < Mb; m++) {
        const size_t r0 = (size_t)(k0 + m) * T;
        for (int t = tid; t < T; t += kThreads) alS[t] = a.act_lz[(r0 + t) * 2] - log(a.act_lz[(r0 + t) * 2 + 1]);
        __syncthreads();
        if (tid == 0) {
            double lp = 0.0;
            for (int t = 0; t < T; t++) lp += alS[t];
            a.logp[k0 + m] = lp;
        }
        __syncthreads();
    }
}

}  // namespace dp


using namespace dp;

// ---------------------------------------------------------------- host API
static ParamLayout layout_of(int V1, int D, int dd, int F, int td) {
    ParamLayout o;
    int64_t p = 0;
    o.type_table = p;
    p += (int64_t)V1 * td;
    o.dev_table = p;
    p += (int64_t)(D + 1) * dd;
    o.w_enc = p;
    p += (int64_t)(F + kH) * kG;
    o.b_enc = p;
    p += kG;
    o.w_dec = p;
    p += (int64_t)(dd + kH) * kG;
    o.b_dec = p;
    p += kG;
    o.w_att = p;
    p += (int64_t)kH * kH;
    o.w_out = p;
    p += (int64_t)2 * kH * dd;
    o.b_out = p;
    p += D;
    o.total = p;
    return o;
}

extern "C" void dp_policy_destroy(dp_policy *p) {
    if (!p) return;
    void *ptrs[] = {p->type_off, p->type_idx, p->occ_off, p->occ_t, p->zeros, p->shape, p->adj, p->X, p->XP, p->enc_h, p->enc_c,
                    p->enc_g, p->edev, p->act_h, p->act_c, p->act_g, p->act_uc, p->row_du, p->proj, p->encW, p->proj_nmax, p->vdev, p->act_u, p->act_p,
                    p->act_stat, p->act_lz, p->act_choice, p->act_logp, p->row_q, p->row_w,
                    p->row_dq, p->row_dhx, p->dh0, p->dc0, p->d_enc, p->gsum, p->da_enc, p->partial, p->gacc,
                    p->tile_part, p->tile_partA, p->partA, p->a_tot, p->act_e, p->act_esc, p->da_colexp, p->proj_dig, p->proj_inv};
    for (void *q : ptrs)
        if (q) cudaFree(q);
    if (p->side) cudaStreamDestroy(p->side);
    if (p->side2) cudaStreamDestroy(p->side2);
    if (p->ev_fork) cudaEventDestroy(p->ev_fork);
    if (p->ev_join) cudaEventDestroy(p->ev_join);
    if (p->ev_fork2) cudaEventDestroy(p->ev_fork2);
    if (p->ev_join2) cudaEventDestroy(p->ev_join2);
    if (p->ev_att) cudaEventDestroy(p->ev_att);
    if (p->ev_rows) cudaEventDestroy(p->ev_rows);
    (void)cudaGetLastError();
    delete p;
}

size_t dp_backward_partial_elems(const dp_policy *p);  // policy_bwd.cu

extern "C" int dp_policy_create(int32_t T, int32_t n_dev, int32_t hidden, int32_t dev_dim, int32_t type_dim,
                                int32_t shape_slots, int32_t adj_slots, int32_t vocab_rows,
                                const int32_t *h_type_off, const int32_t *h_type_idx, const double *h_shape,
                                const double *h_adj, int32_t k_max, dp_policy **out) {
    DP_ENTRY();
    DP_REQUIRE(out != nullptr, "dp_policy_create: out is NULL");
    DP_REQUIRE(T >= 1, "cannot place an empty group sequence");
    DP_REQUIRE(hidden == kH, "dp_policy_create: this build supports hidden=64 (reference default)");
    DP_REQUIRE(n_dev >= 1 && n_dev <= kMaxD, "dp_policy_create: need 1 <= num_devices <= 32");
    DP_REQUIRE(dev_dim >= 1 && dev_dim <= kMaxDD, "dp_policy_create: need 1 <= dev_dim <= 32");
    DP_REQUIRE(type_dim >= 1 && shape_slots >= 1 && adj_slots >= 1, "all embedding widths must be >= 1");
    DP_REQUIRE(vocab_rows >= 1 && k_max >= 1, "dp_policy_create: bad vocab_rows / k_max");
    dp_policy *p = new dp_policy();
    PolicyDims &dm = p->dims;
    dm.T = T;
    dm.D = n_dev;
    dm.dd = dev_dim;
    dm.td = type_dim;
    dm.ss = shape_slots;
    dm.as = adj_slots;
    dm.F = type_dim + shape_slots + adj_slots;
    dm.V1 = vocab_rows;
    dm.off = layout_of(vocab_rows, n_dev, dev_dim, dm.F, type_dim);
    p->k_max = k_max;
    const int n_idx = h_type_off[T];
    for (int t = 0; t < T; t++)
        if (h_type_off[t + 1] <= h_type_off[t]) {
            dp_policy_destroy(p);
            dp::set_error("dp_policy_create: every group needs >= 1 member type");
            return DP_EINVAL;
        }
    const size_t rows = (size_t)k_max * T;
    bool ok = true;
    auto alloc = [&](void **dst, size_t bytes) {
        if (!ok) return;
        if (cudaMalloc(dst, bytes ? bytes : 8) != cudaSuccess) ok = false;
    };
    auto upload = [&](void **dst, const void *src, size_t bytes) {
        alloc(dst, bytes);
        if (ok && bytes && cudaMemcpy(*dst, src, bytes, cudaMemcpyHostToDevice) != cudaSuccess) ok = false;
    };
    upload((void **)&p->type_off, h_type_off, sizeof(int32_t) * (T + 1));
    upload((void **)&p->type_idx, h_type_idx, sizeof(int32_t) * n_idx);
    {
        std::vector<int32_t> occ_off(vocab_rows + 1, 0), occ_t(n_idx);
        for (int i = 0; i < n_idx; i++) {
            if (h_type_idx[i] < 0 || h_type_idx[i] >= vocab_rows) {
                dp_policy_destroy(p);
                dp::set_error("dp_policy_create: type index out of range");
                return DP_EINVAL;
            }
            occ_off[h_type_idx[i] + 1]++;
        }
        for (int v = 0; v < vocab_rows; v++) occ_off[v + 1] += occ_off[v];
        std::vector<int32_t> fill(occ_off.begin(), occ_off.end() - 1);
        for (int t = 0; t < T; t++)
            for (int i = h_type_off[t]; i < h_type_off[t + 1]; i++) occ_t[fill[h_type_idx[i]]++] = t;
        upload((void **)&p->occ_off, occ_off.data(), sizeof(int32_t) * (vocab_rows + 1));
        upload((void **)&p->occ_t, occ_t.data(), sizeof(int32_t) * n_idx);
        p->n_occ = n_idx;
        std::vector<double> z(kH, 0.0);
        upload((void **)&p->zeros, z.data(), sizeof(double) * kH);
    }
    upload((void **)&p->shape, h_shape, sizeof(double) * T * shape_slots);
    upload((void **)&p->adj, h_adj, sizeof(double) * T * adj_slots);
    alloc((void **)&p->X, sizeof(double) * T * dm.F);
    alloc((void **)&p->XP, sizeof(double) * T * kG);
    alloc((void **)&p->enc_h, sizeof(double) * T * kH);
    alloc((void **)&p->enc_c, sizeof(double) * T * kH);
    alloc((void **)&p->enc_g, sizeof(double) * T * kG);
    alloc((void **)&p->edev, sizeof(double) * (n_dev + 1) * kG);
    alloc((void **)&p->act_h, sizeof(double) * rows * kH);
    alloc((void **)&p->act_c, sizeof(double) * rows * kH);
    alloc((void **)&p->act_g, sizeof(double) * rows * kG);
    alloc((void **)&p->act_uc, sizeof(double) * rows * dev_dim);
    alloc((void **)&p->row_du, sizeof(double) * rows * dev_dim);
    alloc((void **)&p->proj, sizeof(double) * T * kH);
    alloc((void **)&p->encW, sizeof(double) * T * dev_dim);
    alloc((void **)&p->proj_nmax, sizeof(unsigned long long));
    alloc((void **)&p->vdev, sizeof(double) * kH * n_dev);
    alloc((void **)&p->act_u, sizeof(double) * rows * dev_dim);
    alloc((void **)&p->act_p, sizeof(double) * rows * n_dev);
    alloc((void **)&p->act_stat, sizeof(double) * rows * 2);
    alloc((void **)&p->act_lz, sizeof(double) * rows * 2);
    alloc((void **)&p->act_choice, rows);
    alloc((void **)&p->act_logp, sizeof(double) * k_max);
    alloc((void **)&p->row_q, sizeof(double) * rows * kH);
    alloc((void **)&p->row_w, sizeof(double) * rows);
    alloc((void **)&p->row_dq, sizeof(double) * rows * kH);
    alloc((void **)&p->row_dhx, sizeof(double) * rows * kH);
    alloc((void **)&p->dh0, sizeof(double) * k_max * kH);
    alloc((void **)&p->dc0, sizeof(double) * k_max * kH);
    alloc((void **)&p->d_enc, sizeof(double) * T * kH);
    alloc((void **)&p->gsum, sizeof(double) * T * kH);
    alloc((void **)&p->da_enc, sizeof(double) * T * kG);
    alloc((void **)&p->da_colexp, sizeof(int) * kG);
    alloc((void **)&p->proj_dig, att_bwd_tc_proj_bytes(T));
    alloc((void **)&p->proj_inv, sizeof(double) * kH);
    p->partial_elems = dp_backward_partial_elems(p);
    alloc((void **)&p->partial, sizeof(double) * p->partial_elems);
    alloc((void **)&p->gacc, sizeof(double) * dm.off.total);
    // split backward (rows half overlapping the simulator) keeps one T x 64
    // d_enc partial per (sample, 64-step tile): K*T^2*8 bytes — allocated only
    // below 2 GiB (134 MB at C3 K=256; C5 K=4096 would need 134 GB and uses
    // the fused pass)
    const size_t tiles = (size_t)k_max * ((T + 63) / 64);
    const size_t part_bytes = sizeof(double) * tiles * (size_t)T * kH;
    if (ok && part_bytes <= (size_t)2 << 30) {
        alloc((void **)&p->tile_part, part_bytes);
        alloc((void **)&p->tile_partA, sizeof(double) * tiles * (size_t)T * dev_dim);
    }
    alloc((void **)&p->partA, sizeof(double) * 2 * kNumSMs * (size_t)T * dev_dim);
    // stored attention numerators (the backward skips the score recompute): K*T^2*8 bytes,
    // kept below 2 GiB (134 MB at C3 K=256)
    if (ok && sizeof(double) * rows * (size_t)T <= ((size_t)2 << 30)) {
        alloc((void **)&p->act_e, sizeof(double) * rows * (size_t)T);
        alloc((void **)&p->act_esc, sizeof(double) * rows * kWarps);
    }
    alloc((void **)&p->a_tot, sizeof(double) * (size_t)T * dev_dim);
    if (!ok) {
        dp::set_error(std::string("dp_policy_create: allocation/upload failed: ") +
                      cudaGetErrorString(cudaGetLastError()));
        dp_policy_destroy(p);
        return DP_ECUDA;
    }
    if (cudaStreamCreateWithFlags(&p->side, cudaStreamNonBlocking) != cudaSuccess ||
        cudaStreamCreateWithFlags(&p->side2, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&p->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&p->ev_join, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&p->ev_fork2, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&p->ev_join2, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&p->ev_att, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&p->ev_rows, cudaEventDisableTiming) != cudaSuccess) {
        dp::set_error("dp_policy_create: stream/event creation failed");
        dp_policy_destroy(p);
        return DP_ECUDA;
    }
    p->last_K = 0;
    *out = p;
    return DP_OK;
}

extern "C" int64_t dp_policy_num_params(const dp_policy *p) { return p ? p->dims.off.total : -1; }

// Debug: enable (1) / disable (0) decoder phase clocks, then read and reset
// the 8 per-phase cycle sums (block 0) into h_out[8].  Synchronous.
static int g_enc_variant = 0;  // dp_debug_encoder_variant
// Debug: encoder recurrence kernel (0 = one CTA, 1 = 4-CTA cluster with a DSMEM h exchange)
extern "C" int dp_debug_encoder_variant(int32_t mode) {
    DP_ENTRY();
    DP_REQUIRE(mode == 0 || mode == 1, "dp_debug_encoder_variant: mode must be 0 or 1");
    g_enc_variant = mode;
    return DP_OK;
}
static int g_dec_variant = 0;  // dp_debug_decoder_variant
static bool g_clocks_on = false;  // dp_debug_phase_clocks: launch the CLK instantiations
extern "C" int dp_debug_decoder_variant(int32_t mode) {
    DP_ENTRY();
    DP_REQUIRE(mode >= 0 && mode <= 5, "dp_debug_decoder_variant: mode must be 0..5");
    g_dec_variant = mode;
    return DP_OK;
}

// Debug: free the optional backward stores so a small engine takes the code
// paths a C5-sized one does (mask bit 0: attention numerators act_e/act_esc ->
// score-recompute att_bwd<false>; bit 1: per-tile partials tile_part/A -> the
// rows pass is skipped and the grads call runs the fused backward).
extern "C" int dp_debug_policy_drop_stores(dp_policy *p, int32_t mask) {
    DP_ENTRY();
    DP_REQUIRE(p, "dp_debug_policy_drop_stores: NULL policy");
    DP_CUDA_TRY(cudaDeviceSynchronize());
    auto drop = [](double *&q) {
        if (q) cudaFree(q);
        q = nullptr;
    };
    if (mask & 1) {
        drop(p->act_e);
        drop(p->act_esc);
    }
    if (mask & 2) {
        drop(p->tile_part);
        drop(p->tile_partA);
    }
    p->rows_ready = 0;
    return DP_OK;
}

extern "C" int dp_debug_phase_clocks(int32_t enable, int64_t *h_out) {
    DP_ENTRY();
    const int on = enable ? 1 : 0;
    {
        const int skip = enable > 1 ? enable >> 1 : 0;  // debug ablation bits (enable = 1 | skip << 1)
        DP_CUDA_TRY(cudaMemcpyToSymbol(g_dbg_skip, &skip, sizeof(int)));
    }
    DP_CUDA_TRY(cudaMemcpyToSymbol(g_dbg_clocks, &on, sizeof(int)));
    g_clocks_on = on != 0;
    if (h_out) DP_CUDA_TRY(cudaMemcpyFromSymbol(h_out, g_phase_clk, sizeof(long long) * 16));
    long long z[16] = {0};
    DP_CUDA_TRY(cudaMemcpyToSymbol(g_phase_clk, z, sizeof(z)));
    return DP_OK;
}

// Debug: read and reset the decoder's per-warp phase-end arrival sums (block 0,
// cycles from the phase start summed over steps) into h_out[8 * 3] (warp-major).
extern "C" int dp_debug_warp_clocks(int64_t *h_out) {
    DP_ENTRY();
    DP_REQUIRE(h_out, "dp_debug_warp_clocks: NULL argument");
    DP_CUDA_TRY(cudaMemcpyFromSymbol(h_out, g_warp_clk, sizeof(long long) * kWarps * 3));
    long long z[kWarps * 3] = {0};
    DP_CUDA_TRY(cudaMemcpyToSymbol(g_warp_clk, z, sizeof(z)));
    return DP_OK;
}

extern "C" int dp_policy_read_inputs(const dp_policy *p, double *out, void *stream) {
    DP_ENTRY();
    DP_REQUIRE(p && out, "dp_policy_read_inputs: NULL argument");
    DP_CUDA_TRY(cudaMemcpyAsync(out, p->X, sizeof(double) * p->dims.T * p->dims.F, cudaMemcpyDeviceToDevice,
                                (cudaStream_t)stream));
    return DP_OK;
}

extern "C" int dp_policy_encode(dp_policy *p, const double *params, void *stream) {
    DP_ENTRY();
    DP_REQUIRE(p && params, "dp_policy_encode: NULL argument");
    cudaStream_t st = (cudaStream_t)stream;
    const PolicyDims &dm = p->dims;
    DP_REQUIRE(dm.F <= 512 && dm.dd <= 512, "dp_policy_encode: input width above 512");
    enc_prologue_kernel<<<dm.T + dm.D + 1, kG, 0, st>>>(dm, params, p->type_off, p->type_idx, p->shape, p->adj, p->X,
                                                       p->XP, p->edev);
    DP_LAUNCH_CHECK();
    if (g_clocks_on)
        enc_rec_kernel<true><<<1, kThreads, 0, st>>>(dm, params, p->XP, p->enc_h, p->enc_c, p->enc_g);
    else if (g_enc_variant == 1)
        enc_rec_cluster_kernel<<<kEncCl, kThreads, 0, st>>>(dm, params, p->XP, p->enc_h, p->enc_c, p->enc_g);
    else
        enc_rec_kernel<false><<<1, kThreads, 0, st>>>(dm, params, p->XP, p->enc_h, p->enc_c, p->enc_g);
    DP_LAUNCH_CHECK();
    DP_CUDA_TRY(cudaMemsetAsync(p->proj_nmax, 0, sizeof(unsigned long long), st));
    dec_prep_kernel<<<dm.T, 128, 0, st>>>(dm, params, p->enc_h, p->proj, p->encW, p->proj_nmax, p->vdev);
    DP_LAUNCH_CHECK();
    return DP_OK;
}

namespace {
struct DecPlan {
    int M, MT, enc_in_smem, spec, tcg, Tpad;
    size_t smem;
    DecArgs proto;
};

bool plan_decoder(const PolicyDims &dm, int K, int variant_mode, DecPlan &pl) {
    const int T = dm.T, D = dm.D, dd = dm.dd;
    const size_t budget = 225 * 1024;
    // M = samples per CTA, a power of two (== the kernel's MT: the per-sample
    // loops run branch-free over all MT slots)
    int M = ceil_div(K, kNumSMs);
    M = M <= 1 ? 1 : M <= 2 ? 2 : M <= 4 ? 4 : 8;
    for (; M >= 1; M >>= 1) {
        const int MT = M;
        // preference: proj in smem + speculative cell, proj in smem, global proj (+spec), global
        for (int variant = 0; variant < 4; variant++) {
            // the speculative cell costs D x the gate transcendentals on 8-M warps:
            // measured slower at C3 (D=4, M=2), so it is opt-in (mode 1)
            const int enc_smem = variant < 2, spec = (variant % 2 == 0) && MT <= 4 && variant_mode == 1;
            if (variant % 2 == 0 && !spec) continue;
            DecArgs &a = pl.proto;
            // tensor-core gates (TCG) on the FAST path: opt-in (mode 4).  Measured at C3
            // (M=2, per-step phase clocks, same run): fp64 gates A 1321 / C 3989 / E 1914
            // cycles; TCG A 1830 / C 3414 / E 2078 — the scores-only pass saves 1.1K cycles
            // in C but the MMAs' operand traffic (+550 in C), the accumulator read-back
            // (+250 in A) and the digit stores (+140 in A) give it back
            const int tcg = enc_smem && !spec && MT <= 2 && D <= 4 && dd <= 16 && T <= kThreads && variant_mode == 4;
            // score rows [M][Tpad] with Tpad == 4 (mod 16) doubles: the DM path's
            // fragment loads (8 samples x 4 rows) hit distinct banks
            const int Tpad = ((T + 11) & ~15) + 4;
            int o = 0;
            auto take = [&](int n) {
                const int r = o;
                o += (n + 1) & ~1;
                return r;
            };
            a.o_proj = enc_smem && !tcg ? take(T * kProjLd) : 0;
            a.ewld = ((T + 1) & ~1) + 2;
            a.o_encw = enc_smem ? take(a.ewld * dd) : 0;
            a.o_wout = take(kWout1Ld * dd);
            a.o_devt = take(D * dd);
            a.o_bout = take(D);
            a.o_edev = spec ? 0 : take((D + 1) * kG);
            a.o_h = spec ? 0 : take(M * kH);
            a.o_uh = take(M * 32);
            a.o_alpha = take(std::max(M * (Tpad > kH ? Tpad : kH),
                                      MT == 8 && !enc_smem ? kWarps * kDmsSlots * kDmsSlot : 0));
            a.o_pm = take(kWarps * M);
            a.o_ps = take(kWarps * M);
            a.o_puc = take(kWarps * M * dd);
            a.o_pz = take(kWarps * M * D);
            a.o_gn = spec ? take(M * kG) : 0;
            a.o_hc = spec ? take(M * D * kH) : 0;
            a.o_cc = spec ? take(2 * M * D * kH) : 0;
            a.o_ac = spec ? take(M * D * kG) : 0;
            a.o_pcg = take(2 * M);
            a.o_misc = take(16 + 2 * M);
            a.o_rn = take(2 * M);
            a.o_fin = take(49 * M);  // FAST: [2][M][16 or 24] step records + [M] running sampling margins
            a.o_v = take(kH * D);
            a.o_wo = take(kH * dd);
            if (tcg) {
                o = (o + 15) & ~15;  // 128-byte aligned B operands
                a.o_bdig = take(2 * 11 * 256 / 8);
                a.o_tmb = take(2);
            } else {
                a.o_bdig = a.o_tmb = 0;
            }
            const size_t bytes = (size_t)o * sizeof(double);
            if (bytes <= budget) {
                pl.M = M;
                pl.MT = MT;
                pl.enc_in_smem = enc_smem;
                pl.spec = spec;
                pl.tcg = tcg;
                pl.Tpad = Tpad;
                pl.smem = bytes;
                return true;
            }
        }
        if (M == 1) break;
    }
    return false;
}

template <bool PS, bool SPEC>
const void *dec_fn(int MT, bool fast, bool tcg, bool fast8 = false) {
    if constexpr (PS && !SPEC) {
        if (fast8)  // FAST with 4 < D <= 8 devices
            return g_clocks_on ? (MT == 1   ? (const void *)dec_kernel<1, PS, false, true, false, true, 8>
                                  : MT == 2 ? (const void *)dec_kernel<2, PS, false, true, false, true, 8>
                                            : (const void *)dec_kernel<4, PS, false, true, false, true, 8>)
                               : (MT == 1   ? (const void *)dec_kernel<1, PS, false, true, false, false, 8>
                                  : MT == 2 ? (const void *)dec_kernel<2, PS, false, true, false, false, 8>
                                            : (const void *)dec_kernel<4, PS, false, true, false, false, 8>);
        if (fast && tcg)
            return g_clocks_on ? (MT == 1 ? (const void *)dec_kernel<1, PS, false, true, true, true>
                                          : (const void *)dec_kernel<2, PS, false, true, true, true>)
                               : (MT == 1 ? (const void *)dec_kernel<1, PS, false, true, true>
                                          : (const void *)dec_kernel<2, PS, false, true, true>);
        if (fast)
            return g_clocks_on ? (MT == 1   ? (const void *)dec_kernel<1, PS, false, true, false, true>
                                  : MT == 2 ? (const void *)dec_kernel<2, PS, false, true, false, true>
                                            : (const void *)dec_kernel<4, PS, false, true, false, true>)
                               : (MT == 1   ? (const void *)dec_kernel<1, PS, false, true>
                                  : MT == 2 ? (const void *)dec_kernel<2, PS, false, true>
                                            : (const void *)dec_kernel<4, PS, false, true>);
    }
    if constexpr (!PS && !SPEC) {
        if (MT == 8 && g_clocks_on) return (const void *)dec_kernel<8, PS, false, false, false, true>;
    }
    if constexpr (PS && !SPEC) {
        if (MT == 4 && g_clocks_on) return (const void *)dec_kernel<4, PS, false, false, false, true>;
    }
    if (SPEC)
        return MT == 1 ? (const void *)dec_kernel<1, PS, SPEC>
               : MT == 2 ? (const void *)dec_kernel<2, PS, SPEC>
                         : (const void *)dec_kernel<4, PS, SPEC>;
    return MT == 1 ? (const void *)dec_kernel<1, PS, false>
           : MT == 2 ? (const void *)dec_kernel<2, PS, false>
           : MT == 4 ? (const void *)dec_kernel<4, PS, false>
                     : (const void *)dec_kernel<8, PS, false>;
}
}  // namespace

// Debug / tests: the decoder plan for a batch of K on this engine:
// out[6] = {samples per CTA, kernel MT, tensor-core gates, shared-memory bytes,
// speculative cell, operands in shared memory}.
extern "C" int dp_debug_decoder_plan(const dp_policy *p, int32_t K, int32_t *out) {
    DP_ENTRY();
    DP_REQUIRE(p && out && K >= 1, "dp_debug_decoder_plan: bad arguments");
    DecPlan pl;
    DP_REQUIRE(plan_decoder(p->dims, K, g_dec_variant, pl), "dp_debug_decoder_plan: shared-memory plan failed");
    const bool fast = pl.MT <= 2 && p->dims.D <= 4 && p->dims.dd <= 16 && p->dims.T <= kThreads;
    out[0] = pl.M;
    out[1] = pl.MT;
    out[2] = pl.tcg && fast && pl.enc_in_smem && !pl.spec;
    out[3] = (int32_t)pl.smem;
    out[4] = pl.spec;
    out[5] = pl.enc_in_smem;
    return DP_OK;
}

extern "C" int dp_policy_decode(dp_policy *p, const double *params, int32_t K, int64_t k_offset,
                                const uint64_t *h_pcg, uint64_t draw_base, const int64_t *draw_counter,
                                int64_t draws_per_count, const uint8_t *forced, uint8_t *choice_out,
                                double *logp, double *probs_out, double *margin, void *stream) {
    DP_ENTRY();
    DP_REQUIRE(p && params && logp, "dp_policy_decode: NULL argument");
    DP_REQUIRE(K >= 1 && K <= p->k_max, "dp_policy_decode: K out of range (1..k_max)");
    DP_REQUIRE(forced || h_pcg, "dp_policy_decode: need a PCG64 state or a forced placement");
    const PolicyDims &dm = p->dims;
    DecPlan pl;
    DP_REQUIRE(plan_decoder(dm, K, g_dec_variant, pl), "dp_policy_decode: shared-memory plan failed");
    DecArgs a = pl.proto;
    a.dm = dm;
    a.params = params;
    a.K = K;
    a.k_offset = k_offset;
    if (h_pcg) {
        a.st_hi = h_pcg[0];
        a.st_lo = h_pcg[1];
        a.inc_hi = h_pcg[2];
        a.inc_lo = h_pcg[3];
    } else {
        a.st_hi = a.st_lo = a.inc_hi = a.inc_lo = 0;
    }
    a.draw_base = draw_base;
    a.draw_counter = (const long long *)draw_counter;
    a.draws_per_count = draws_per_count;
    a.forced = forced;
    a.enc_h = p->enc_h;
    a.enc_c = p->enc_c;
    a.edev = p->edev;
    a.proj = p->proj;
    a.encW = p->encW;
    a.proj_nmax = p->proj_nmax;
    a.vdev = p->vdev;
    a.act_h = p->act_h;
    a.act_c = p->act_c;
    a.act_g = p->act_g;
    a.act_uc = p->act_uc;
    a.act_e = p->act_e;
    a.act_esc = p->act_esc;
    a.act_u = p->act_u;
    a.act_p = p->act_p;
    a.act_stat = p->act_stat;
    a.act_lz = p->act_lz;
    a.choice = p->act_choice;
    a.choice_out = choice_out;
    a.logp = logp;
    a.probs_out = probs_out;
    a.margin = forced ? nullptr : margin;
    a.M = pl.M;
    a.Tpad = pl.Tpad;
    a.ewld = ((dm.T + 1) & ~1) + 2;
    const int grid = ceil_div(K, pl.M);
    cudaStream_t st = (cudaStream_t)stream;
    // FAST: compact instantiation for <= 4 samples per CTA (debug mode 5: the generic kernel
    // for 4 samples per CTA, A/B)
    const bool fast = (pl.MT <= 2 || (pl.MT == 4 && g_dec_variant != 5)) && dm.D <= 4 && dm.dd <= 16 &&
                      dm.T <= kThreads;
    // ... and its instantiation for 4 < D <= 8 devices (C2's 4 GPUs + CPU)
    const bool fast8 = pl.MT <= 4 && g_dec_variant != 5 && dm.D > 4 && dm.D <= 8 && dm.dd <= 16 &&
                       dm.T <= kThreads && !pl.tcg;
    const void *fn = pl.enc_in_smem
                         ? (pl.spec ? dec_fn<true, true>(pl.MT, false, false)
                                    : dec_fn<true, false>(pl.MT, fast, pl.tcg, fast8))
                         : (pl.spec ? dec_fn<false, true>(pl.MT, false, false) : dec_fn<false, false>(pl.MT, false, false));
    DP_CUDA_TRY(allow_big_smem(fn, pl.smem));
    void *args[] = {&a};
    DP_CUDA_TRY(cudaLaunchKernel(fn, dim3(grid), dim3(kThreads), args, pl.smem, st));
    count_launch();
    p->last_K = K;
    p->rows_ready = 0;
    return DP_OK;
}
