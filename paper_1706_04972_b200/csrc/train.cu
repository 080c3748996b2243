// REINFORCE epilogue and Adam on sm_100a: everything after scoring, on device,
// so one training update is a fixed launch sequence (CUDA-graph capturable).
//
// Reference (/root/reference/pkg/src/devplace/trainer.py):
//   reward_of            66-72     R = sqrt(m) | failing signal
//   best-so-far          284-287   strict <, feasible only, k order
//   success-only filter  289-292
//   reinforce_update     138-154   adv = R - B over used samples; /= n_used
//   BaselineState.update 83-84     B <- decay*B + (1-decay)*mean(used R)
//   LogRow               298-308   mean_R = np.mean(all K rewards)
//   ParameterStore.apply 113-131   finite check, Adam, version++
// Scalar statistics replicate numpy's pairwise summation exactly and the
// Adam element recurrences use unfused mul/add in numpy's order (compiled
// with --fmad=false), so logs and the optimizer match bit-for-bit given an
// identical gradient.

#include <math.h>

#include "policy.cuh"

namespace dp {
namespace {

// numpy pairwise_sum (np.add.reduce / np.mean on a contiguous float64 array):
// blocks of <= 128 summed with 8 interleaved accumulators, larger ranges split
// at n/2 rounded down to a multiple of 8 — restated with an explicit stack
// (device recursion overflowed the default thread stack at K = 4096).
__device__ double np_pairwise_leaf(const double *a, int n) {
    if (n < 8) {
        double r = 0.0;
        for (int i = 0; i < n; i++) r += a[i];
        return r;
    }
    double r[8];
    for (int j = 0; j < 8; j++) r[j] = a[j];
    int i = 8;
    for (; i < n - (n % 8); i += 8)
        for (int j = 0; j < 8; j++) r[j] += a[i + j];
    double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; i++) res += a[i];
    return res;
}

__device__ double np_pairwise(const double *a, int n) {
    constexpr int kDepth = 32;
    int off[kDepth], len[kDepth], stage[kDepth];
    double left[kDepth];
    int sp = 0;
    off[0] = 0;
    len[0] = n;
    stage[0] = 0;
    double ret = 0.0;
    for (;;) {
        const int m = len[sp];
        if (m <= 128 || stage[sp] == 2) {
            ret = m <= 128 ? np_pairwise_leaf(a + off[sp], m) : left[sp] + ret;
            if (sp == 0) return ret;
            sp--;
            continue;
        }
        int n2 = m / 2;
        n2 -= n2 % 8;
        if (stage[sp] == 0) {
            stage[sp] = 1;
            off[sp + 1] = off[sp];
            len[sp + 1] = n2;
        } else {  // left half done
            left[sp] = ret;
            stage[sp] = 2;
            off[sp + 1] = off[sp] + n2;
            len[sp + 1] = m - n2;
        }
        sp++;
        stage[sp] = 0;
    }
}

// single CTA: the block forms the rewards (global loads + sqrt) in parallel,
// then thread 0 runs the order-dependent scalar logic over shared memory
__global__ void epilogue_kernel(int K, int T, const double *__restrict__ makespan,
                                const uint8_t *__restrict__ feasible, const uint8_t *__restrict__ choice,
                                int choice_div, double failing, double decay, long long success_only_after, long long k_offset,
                                int K_local, dp_train_state *st, double *__restrict__ adv,
                                uint8_t *__restrict__ best_choice, double *__restrict__ log_rows, long long log_cap,
                                int controller_id) {
    extern __shared__ double R[];   // [K] rewards, [K] used rewards, [K] feasibility bytes
    __shared__ int s_best_k;
    const int tid = threadIdx.x;
    double *used_r = R + K;
    uint8_t *okS = reinterpret_cast<uint8_t *>(R + 2 * K);
    for (int k = tid; k < K; k += blockDim.x) {
        const bool ok = feasible[k] != 0;
        const double m = makespan[k];
        if (ok && (!isfinite(m) || m <= 0.0)) st->error = 1;  // reward_of raises ValueError
        R[k] = ok ? sqrt(m) : failing;
        okS[k] = ok ? 1 : 0;
    }
    __syncthreads();
    if (tid == 0) {
        const long long upd = st->update;
        double best = st->best_r;
        int best_k = -1, n_feas = 0, n_used = 0;
        const bool all = upd < success_only_after;
        for (int k = 0; k < K; k++) {
            const bool ok = okS[k] != 0;
            const double r = R[k];
            n_feas += ok ? 1 : 0;
            if (ok && r < best) {
                best = r;
                best_k = k;
            }
            if (all || ok) used_r[n_used++] = r;
        }
        const double b_old = st->baseline;
        const double mean_r = np_pairwise(R, K) / (double)K;
        double b_new = b_old;
        if (n_used > 0) {
            const double mu = np_pairwise(used_r, n_used) / (double)n_used;
            b_new = decay * b_old + (1.0 - decay) * mu;
        }
        st->baseline = b_new;
        st->baseline_prev = b_old;
        st->n_used = n_used;
        st->n_feasible = n_feas;
        if (best_k >= 0) {
            st->best_r = best;
            st->best_k = best_k;
            st->best_update = upd;
        }
        s_best_k = best_k;
        if (upd < log_cap) {
            double *row = log_rows + upd * 8;
            row[0] = (double)upd;
            row[1] = (double)controller_id;
            row[3] = mean_r;
            row[4] = b_new;
            row[5] = st->best_r;
            row[6] = (double)n_feas;
            row[7] = (double)n_used;
        }
    }
    __syncthreads();
    // advantages for this rank's samples: (R - B_old) if used else 0
    const bool all = st->update < success_only_after;
    const double b_old = st->baseline_prev;
    const bool any = st->n_used > 0;
    for (int k = tid; k < K_local; k += blockDim.x) {
        const long long kg = k_offset + k;
        const bool use = any && (all || okS[kg] != 0);
        adv[k] = use ? R[kg] - b_old : 0.0;
    }
    const int bk = s_best_k;
    if (bk >= 0)
        for (int t = tid; t < T; t += blockDim.x) best_choice[t] = choice[(size_t)(bk / choice_div) * T + t];
}

// measure() with lognormal noise (pkg/simulator.py:218-223): a feasible
// sample's measurement is np.mean(base * factors[1:]) — the factors row of
// (update, k) comes from the host (the reference's own numpy streams,
// pkg/trainer.py:277), the product and numpy's pairwise mean run here.
__global__ void noise_kernel(int K, long long k_offset, int K_total, double *__restrict__ makespan,
                             const uint8_t *__restrict__ feasible, const double *__restrict__ factors,
                             long long n_updates, int n_factors, dp_train_state *st) {
    const long long u = st->update;
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= K) return;
    if (u < 0 || u >= n_updates) {
        st->error = 2;  // noise table exhausted
        return;
    }
    if (!feasible[k]) return;
    const double base = makespan[k];
    const double *f = factors + ((size_t)u * K_total + k_offset + k) * n_factors;
    double prod[64];
    for (int s = 0; s < n_factors; s++) prod[s] = base * f[s];
    makespan[k] = np_pairwise(prod, n_factors) / (double)n_factors;
}

__global__ void finite_check_kernel(long long P, const double *__restrict__ g, int *__restrict__ flag) {
    long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    int bad = 0;
    for (; i < P; i += (long long)gridDim.x * blockDim.x) bad |= !isfinite(g[i]);
    bad = __syncthreads_or(bad);
    if (threadIdx.x == 0 && bad) atomicOr(flag, 1);
}

// numpy order: m = b1*m + (1-b1)*g ; v = b2*v + (1-b2)*g*g ; mh = m/(1-b1^t) ;
// vh = v/(1-b2^t) ; p -= lr*mh / (sqrt(vh) + eps)   (pkg/trainer.py:125-129)
__global__ void adam_kernel(long long P, double *__restrict__ p, double *__restrict__ m, double *__restrict__ v,
                            const double *__restrict__ grad, const double *__restrict__ bias_corr, long long t_cap,
                            double lr, double b1, double b2, double eps, const dp_train_state *st,
                            const dp_train_state *store, const int *__restrict__ flag) {
    const long long nu = st->n_used;
    if (nu <= 0 || *flag) return;
    const long long t = store->adam_t + 1;
    if (t > t_cap) return;  // step_finalize flags it (error 3) and skips the bump
    const double bc1 = bias_corr[2 * (t - 1)], bc2 = bias_corr[2 * (t - 1) + 1];
    const double c1 = 1.0 - b1, c2 = 1.0 - b2;
    const double n = (double)nu;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < P; i += (long long)gridDim.x * blockDim.x) {
        const double g = grad[i] / n;
        const double mi = b1 * m[i] + c1 * g;
        const double vi = b2 * v[i] + c2 * g * g;
        m[i] = mi;
        v[i] = vi;
        const double mh = mi / bc1;
        const double vh = vi / bc2;
        p[i] = p[i] - lr * mh / (sqrt(vh) + eps);
    }
}

__global__ void step_finalize_kernel(dp_train_state *st, dp_train_state *store, int *flag, double *log_rows,
                                     long long log_cap, long long t_cap) {
    if (threadIdx.x != 0) return;
    if (st->n_used > 0) {
        if (!*flag && store->adam_t + 1 > t_cap) {
            st->error = 3;  // bias-correction table exhausted: no silent frozen update
        } else if (*flag) {
            store->rejected += 1;
        } else {
            store->adam_t += 1;
            store->version += 1;
        }
    }
    if (st->update < log_cap) log_rows[st->update * 8 + 2] = (double)store->version;
    *flag = 0;
    st->update += 1;
}

// K-sharded exchange record (include/devplace_b200.h dp_exchange_*): one CTA
// per rank record.  pack: warp-parallel first-minimum of the feasible rewards
// (sqrt, the epilogue's own R), then the record's bytes.
__host__ __device__ inline long long exch_fe_off(int K_local) { return 8LL * K_local; }
__host__ __device__ inline long long exch_row_off(int K_local) { return 8LL * K_local + K_local; }
__host__ __device__ inline long long exch_bytes(int K_local, int T) {
    return (exch_row_off(K_local) + T + 15) / 16 * 16;
}

__global__ void exchange_pack_kernel(int K_local, int T, const double *__restrict__ makespan,
                                     const uint8_t *__restrict__ feasible, const uint8_t *__restrict__ choice,
                                     uint8_t *__restrict__ rec) {
    __shared__ double sr[32];
    __shared__ int sk[32];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
    double best = INFINITY;
    int bk = 0x7fffffff;
    for (int k = tid; k < K_local; k += blockDim.x) {
        const double m = makespan[k];
        reinterpret_cast<double *>(rec)[k] = m;
        const uint8_t ok = feasible[k];
        rec[exch_fe_off(K_local) + k] = ok;
        const double r = sqrt(m);
        if (ok && (r < best || (r == best && k < bk))) {
            best = r;
            bk = k;
        }
    }
    for (int o = 16; o > 0; o >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int ok2 = __shfl_xor_sync(0xffffffffu, bk, o);
        if (ob < best || (ob == best && ok2 < bk)) {
            best = ob;
            bk = ok2;
        }
    }
    if (lane == 0) {
        sr[warp] = best;
        sk[warp] = bk;
    }
    __syncthreads();
    if (tid == 0) {
        for (int w = 1; w < nw; w++)
            if (sr[w] < sr[0] || (sr[w] == sr[0] && sk[w] < sk[0])) {
                sr[0] = sr[w];
                sk[0] = sk[w];
            }
    }
    __syncthreads();
    const int kb = sk[0] < K_local ? sk[0] : 0;  // no feasible sample: any row (never selected)
    for (int t = tid; t < T; t += blockDim.x) rec[exch_row_off(K_local) + t] = choice[(size_t)kb * T + t];
}

__global__ void exchange_unpack_kernel(int K_local, int T, const uint8_t *__restrict__ recs,
                                       double *__restrict__ makespan, uint8_t *__restrict__ feasible,
                                       uint8_t *__restrict__ rows) {
    const int r = blockIdx.x;
    const uint8_t *rec = recs + (size_t)r * exch_bytes(K_local, T);
    for (int k = threadIdx.x; k < K_local; k += blockDim.x) {
        makespan[(size_t)r * K_local + k] = reinterpret_cast<const double *>(rec)[k];
        feasible[(size_t)r * K_local + k] = rec[exch_fe_off(K_local) + k];
    }
    for (int t = threadIdx.x; t < T; t += blockDim.x) rows[(size_t)r * T + t] = rec[exch_row_off(K_local) + t];
}

// Sampling certificate of one decode: running minimum of the
// per-sample margins and the count of samples below tol, in one launch.
__global__ void margin_accumulate_kernel(int K, const double *__restrict__ margin, double tol,
                                         double *__restrict__ margin_min, long long *__restrict__ n_below) {
    __shared__ double smin[32];
    __shared__ int scnt[32];
    double mn = INFINITY;
    int cnt = 0;
    for (int k = threadIdx.x; k < K; k += blockDim.x) {
        const double m = margin[k];
        mn = fmin(mn, m);
        cnt += m < tol ? 1 : 0;
    }
    for (int o = 16; o > 0; o >>= 1) {
        mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
        cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    }
    const int w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    if ((threadIdx.x & 31) == 0) {
        smin[w] = mn;
        scnt[w] = cnt;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int i = 1; i < nw; i++) {
            mn = fmin(mn, smin[i]);
            cnt += scnt[i];
        }
        margin_min[0] = fmin(margin_min[0], mn);
        n_below[0] += cnt;
    }
}

}  // namespace
}  // namespace dp

using namespace dp;

extern "C" int dp_margin_accumulate(int32_t K, const double *margin, double tol, double *margin_min,
                                    int64_t *n_below, void *stream) {
    DP_ENTRY();
    DP_REQUIRE(K >= 1 && margin && margin_min && n_below, "dp_margin_accumulate: bad argument");
    margin_accumulate_kernel<<<1, 256, 0, (cudaStream_t)stream>>>(K, margin, tol, margin_min,
                                                                  (long long *)n_below);
    DP_LAUNCH_CHECK();
    return DP_OK;
}

extern "C" int64_t dp_exchange_record_bytes(int32_t K_local, int32_t T) { return exch_bytes(K_local, T); }

extern "C" int dp_exchange_pack(int32_t K_local, int32_t T, const double *makespan, const uint8_t *feasible,
                                const uint8_t *choice, uint8_t *record, void *stream) {
    DP_ENTRY();
    DP_REQUIRE(K_local >= 1 && T >= 1 && makespan && feasible && choice && record, "dp_exchange_pack: bad argument");
    exchange_pack_kernel<<<1, 256, 0, (cudaStream_t)stream>>>(K_local, T, makespan, feasible, choice, record);
    DP_LAUNCH_CHECK();
    return DP_OK;
}

extern "C" int dp_exchange_unpack(int32_t nranks, int32_t K_local, int32_t T, const uint8_t *records,
                                  double *makespan, uint8_t *feasible, uint8_t *rows, void *stream) {
    DP_ENTRY();
    DP_REQUIRE(nranks >= 1 && K_local >= 1 && T >= 1 && records && makespan && feasible && rows,
               "dp_exchange_unpack: bad argument");
    exchange_unpack_kernel<<<nranks, 256, 0, (cudaStream_t)stream>>>(K_local, T, records, makespan, feasible, rows);
    DP_LAUNCH_CHECK();
    return DP_OK;
}

extern "C" int dp_reinforce_epilogue(int32_t K, int32_t T, const double *makespan, const uint8_t *feasible,
                                     const uint8_t *choice, int32_t choice_div, double failing, double decay,
                                     int64_t success_only_after, int64_t k_offset, int32_t K_local,
                                     dp_train_state *state, double *adv, uint8_t *best_choice, double *log_rows,
                                     int64_t log_cap, int32_t controller_id, void *stream) {
    DP_ENTRY();
    DP_REQUIRE(K >= 1 && K <= 12288, "dp_reinforce_epilogue: need 1 <= K <= 12288");
    DP_REQUIRE(K_local >= 0 && k_offset >= 0 && k_offset + K_local <= K, "dp_reinforce_epilogue: bad shard");
    DP_REQUIRE(makespan && feasible && choice && state && best_choice && log_rows,
               "dp_reinforce_epilogue: NULL argument");
    DP_REQUIRE(choice_div >= 1, "dp_reinforce_epilogue: choice_div must be >= 1");
    const size_t smem = sizeof(double) * 2 * (size_t)K + (size_t)K;
    DP_CUDA_TRY(allow_big_smem((const void *)epilogue_kernel, smem));
    epilogue_kernel<<<1, 256, smem, (cudaStream_t)stream>>>(K, T, makespan, feasible, choice, choice_div, failing,
                                                            decay,
                                                            success_only_after, k_offset, K_local, state, adv,
                                                            best_choice, log_rows, log_cap, controller_id);
    DP_LAUNCH_CHECK();
    return DP_OK;
}

extern "C" int dp_apply_measurement_noise(int32_t K, int64_t k_offset, int32_t K_total, double *makespan,
                                          const uint8_t *feasible, const double *factors, int64_t n_updates,
                                          int32_t n_factors, dp_train_state *state, void *stream) {
    DP_ENTRY();
    DP_REQUIRE(K >= 1 && makespan && feasible && factors && state, "dp_apply_measurement_noise: NULL argument");
    DP_REQUIRE(k_offset >= 0 && k_offset + K <= K_total, "dp_apply_measurement_noise: bad shard");
    DP_REQUIRE(n_factors >= 1 && n_factors <= 64, "dp_apply_measurement_noise: need 1 <= steps-1 <= 64");
    noise_kernel<<<ceil_div(K, 128), 128, 0, (cudaStream_t)stream>>>(K, k_offset, K_total, makespan, feasible,
                                                                       factors, n_updates, n_factors, state);
    DP_LAUNCH_CHECK();
    return DP_OK;
}

extern "C" int dp_adam_apply(int64_t P, double *params, double *m, double *v, const double *grad,
                             const double *bias_corr, int64_t t_cap, double lr, double b1, double b2, double eps,
                             dp_train_state *state, dp_train_state *store_state, int32_t *flag, double *log_rows,
                             int64_t log_cap, void *stream) {
    DP_ENTRY();
    DP_REQUIRE(P >= 1 && params && m && v && grad && bias_corr && state && flag,
               "dp_adam_apply: NULL argument");
    if (!store_state) store_state = state;
    cudaStream_t st = (cudaStream_t)stream;
    const int blocks = ceil_div(P, 256) < 2 * kNumSMs ? ceil_div(P, 256) : 2 * kNumSMs;
    finite_check_kernel<<<blocks, 256, 0, st>>>(P, grad, flag);
    DP_LAUNCH_CHECK();
    adam_kernel<<<blocks, 256, 0, st>>>(P, params, m, v, grad, bias_corr, t_cap, lr, b1, b2, eps, state, store_state,
                                        flag);
    DP_LAUNCH_CHECK();
    step_finalize_kernel<<<1, 32, 0, st>>>(state, store_state, flag, log_rows, log_cap, t_cap);
    DP_LAUNCH_CHECK();
    return DP_OK;
}
