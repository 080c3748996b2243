// Device-resident policy state shared by the forward/backward kernels.
#pragma once
#include "common.cuh"

namespace dp {

constexpr int kH = 64;        // LSTM width (reference default hidden=64, pkg/trainer.py:173)
constexpr int kG = 4 * kH;    // gates per cell (i, f, o, g — pkg/policy.py:224-233)
constexpr int kThreads = 256; // one thread per gate column in the recurrent kernels
constexpr int kMaxDD = 32;    // device-embedding width limit
constexpr int kMaxD = 32;     // device count limit (u8 choices)
constexpr int kEncPad = kH + 1;  // padded row stride of enc_states in shared memory

// Parameter offsets inside the flat vector, canonical _FIELDS order
// (pkg/policy.py:41-42, 136-146, 168-169).
struct ParamLayout {
    int64_t type_table, dev_table, w_enc, b_enc, w_dec, b_dec, w_att, w_out, b_out, total;
};

struct PolicyDims {
    int T, D, dd, td, ss, as, F, V1;
    ParamLayout off;
};

int dp_tensor_core_mode();  // dp_debug_tensor_core: 0 = tcgen05 paths where supported, 1 = DMMA/SIMT only

// tcgen05 / TMA decoder weight gradient (wgrad_tc.cu)
bool dec_wgrad_tc_ok(const PolicyDims &dm);
int launch_dec_wgrad_tc(const PolicyDims &dm, int rows, const double *act_h, const double *enc_h,
                        const uint8_t *choice, const double *da, const int *colexp, const double *adv, int K,
                        double *partial, int *n_chunks, cudaStream_t st);

// tcgen05 / TMA attention backward, GM rows pass (att_tc.cu)
bool att_bwd_tc_ok(const PolicyDims &dm);
size_t att_bwd_tc_proj_bytes(int T);
int launch_att_bwd_tc(const PolicyDims &dm, int K, const double *proj, uint8_t *proj_dig, double *proj_inv,
                      const double *encW, const double *act_h, const double *row_w, const double *row_du,
                      const double *act_e, const double *act_esc, double *tile_part, double *tile_partA,
                      double *row_dhx, int n_cta, cudaStream_t st);

}  // namespace dp

struct dp_policy {
    dp::PolicyDims dims;
    int k_max;
    // features (uploaded once)
    int32_t *type_off, *type_idx;
    int32_t *occ_off, *occ_t;  // per type row: decode steps using it (with multiplicity), t-ascending
    int n_occ;                 // total occurrences (sum of member-type counts)
    double *zeros;             // [64] zero cell state (encoder step 0)
    double *shape, *adj;
    // encoder activations (one sequence, shared by all samples)
    double *X;      // [T*F]   assembled inputs (pkg/policy.py:256-263)
    double *XP;     // [T*G]   X @ w_enc[:F] + b_enc
    double *enc_h;  // [T*H]   enc_states
    double *enc_c;  // [T*H]
    double *enc_g;  // [T*G]   gate activations i,f,o,g
    double *edev;   // [(D+1)*G] dev_table @ w_dec[:dd] + b_dec (decoder input projection)
    // decoder activations, [k][t][...] (the opaque forward cache)
    double *act_h, *act_c, *act_g, *act_u, *act_p, *act_stat;
    double *act_uc;       // [k*T*dd] ctx @ W_out[64:] (the context enters u, and the backward, only through it)
    double *proj, *encW;  // [T*64] enc @ W_att^T, [T*dd] enc @ W_out[64:] (decoder prologue, per snapshot)
    unsigned long long *proj_nmax;  // max_t ||proj_t|| (IEEE bits): the decoder's no-shift softmax test
    double *vdev;                   // [64*D] W_out[:64] @ dev_table[:D]^T (logits' h half)
    double *act_e;        // [k*T][T] attention numerators e_i = exp(s_i - m_w) (NULL: the backward recomputes)
    double *act_esc;      // [k*T][8] per-warp-slice scale exp(m_w - M) / sum: alpha_i = e_i * esc[(i % 256) / 32]
    double *act_lz;       // [k*T*2] (zs[choice], sum exp zs) -> log-prob terms off the critical path
    uint8_t *act_choice;  // [k*T] by rank
    double *act_logp;     // [k]
    int last_K;
    // backward scratch
    double *row_q, *row_w, *row_dq, *row_dhx;  // per (k,t)
    double *row_du;                                      // [k*T*dd] du = dev_table[:D]^T dz
    double *dh0, *dc0;                                   // [k*H]
    double *d_enc;                                       // [T*H]
    double *gsum;                                        // [T*H] GM: sum_k adv_k ds_k^T H_k
    double *da_enc;                                      // [T*G]
    int *da_colexp;                                      // [G] max biased exponent of |da| per gate column (decoder LSTM backward)
    uint8_t *proj_dig;                                   // proj digit planes per 64-position chunk (tcgen05 attention backward)
    double *proj_inv;                                    // [64] 2^-s per proj column
    double *partial;                                     // per-CTA partial sums
    size_t partial_elems;
    double *gacc;                                        // [P] accumulator
    double *tile_part;            // [k*ceil(T/64)][T][64] per-tile d_enc partials (split backward), NULL if too large
    double *tile_partA;           // [k*ceil(T/64)][T][dd] per-tile A = alpha^T du partials (split backward)
    double *partA;                // [2*SMs][T][dd] per-CTA A partials (fused backward)
    double *a_tot;                // [T][dd] A = sum_rows alpha^T du
    int rows_ready;               // K of the last dp_policy_backward_rows (0: none)
    int att_per_sample;           // the last rows pass left per-sample (1) or per-tile (0) partials
    int att_gmode;                // ... holding G = ds^T H (1, grads pass forms d_enc = G W_att) or d_enc (0)
    // side stream: the encoder backward (one CTA) overlaps the decoder weight-gradient GEMM
    cudaStream_t side, side2;
    cudaEvent_t ev_fork, ev_join, ev_fork2, ev_join2;
    cudaEvent_t ev_att, ev_rows;  // rows pass: attention backward done / whole pass done
};
