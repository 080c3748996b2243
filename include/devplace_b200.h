/*
 * devplace_b200 — C-ABI of the B200-native REINFORCE device-placement hot path.
 *
 * The reference (arXiv 1706.04972 artifact, package `devplace`, pure Python +
 * numpy) has no FFI: its "plugin boundary" is the set of module-level
 * functions the trainer looks up at call time:
 *   pkg/trainer.py:250  trainer-global measure()   -> simulate()
 *   pkg/trainer.py:275  policy_mod.forward_sample()
 *   pkg/trainer.py:150  policy_mod.grad_log_prob()
 *   pkg/trainer.py:293  trainer-global reinforce_update()
 * The Python host package (paper_1706_04972_b200) re-exports those names with
 * the reference signatures and calls down into these entry points through
 * ctypes.  Each entry point below cites the reference function it replaces.
 *
 * Conventions
 *   - Every call returns an int status: DP_OK, DP_EINVAL (host raises
 *     ValueError), DP_ECUDA (CUDA error; dp_last_error() has the text).
 *   - Pointers named h_* are HOST memory read during the call; all other
 *     array pointers are DEVICE memory owned by the caller.
 *   - `stream` is a cudaStream_t (NULL = legacy default stream).  All work is
 *     enqueued on it; no call synchronises unless stated.
 *   - Groups are addressed by topological rank r (gg.topo[r] is the group id,
 *     pkg/graph.py:235-238); the policy's decode step t IS rank t
 *     (pkg/policy.py:99, 310), so placements "by rank" are the decoder's
 *     native output.  Placements "by gid" are the reference's list layout.
 *   - All time / probability arithmetic is IEEE fp64, as in the reference.
 */
#ifndef DEVPLACE_B200_H
#define DEVPLACE_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DP_OK 0
#define DP_EINVAL 1
#define DP_ECUDA 2
#define DP_ECOMM 3

typedef struct dp_graph dp_graph;
typedef struct dp_policy dp_policy;

/* Text of the last error raised on this thread ("" if none). */
const char *dp_last_error(void);

/* Number of kernel launches this library has enqueued (process-wide). */
int64_t dp_launch_count(void);

/* fp64 FMA throughput probe: blocks x threads threads each run 8 independent
 * DFMA chains of `iters` steps (16*iters FLOP per thread).  Used by bench.py
 * to measure the fp64 roofline denominator on the box. */
int dp_fp64_fma_probe(int32_t blocks, int32_t threads, int32_t iters, double *scratch, void *stream);

/* ------------------------------------------------------------------ graph */

/* Upload a grouped graph + device topology (one-time, synchronous).
 * Replaces the per-call setup of simulate(), pkg/simulator.py:122-144:
 * rank (gg.topo_rank), pending counts (len(in_groups)), out-edges sorted by
 * destination rank, per-group cost, plus the check_memory() inputs
 * (pkg/simulator.py:93-106: param_bytes + out_bytes per group).
 *   h_cost[n]       group compute_cost, by rank
 *   h_indeg[n]      distinct predecessor groups, by rank
 *   h_out_off[n+1]  CSR row offsets over out-edges, by source rank
 *   h_out_dst[E]    destination rank, ascending within each row
 *   h_out_bytes[E]  edge tensor_bytes (>= 0)
 *   h_resident[n]   param_bytes + out_bytes, by rank
 *   h_gid[n]        group id of rank r (gg.topo)
 *   h_rate[d], h_bw[d*d] (row = source device), h_mem[d]
 * Limits: n < 65536, 1 <= d <= 32. */
int dp_graph_create(int32_t n, int32_t d, const double *h_cost, const int32_t *h_indeg,
                    const int32_t *h_out_off, const int32_t *h_out_dst, const int64_t *h_out_bytes,
                    const int64_t *h_resident, const int32_t *h_gid, const double *h_rate,
                    const double *h_bw, const int64_t *h_mem, dp_graph **out);
void dp_graph_destroy(dp_graph *g);

/* Score K placements — batched simulate() + check_memory()
 * (pkg/simulator.py:93-106, 122-194; measure() with noise off,
 * pkg/simulator.py:205-219).  One warp per placement (device state in the
 * lanes; one thread per placement for many placements of small graphs — the
 * planner picks), event-exact: makespan/busy/transfer/peak/feasible and the dispatch order are bit-identical
 * to the reference.
 *   placement[K*n]  device ids (u8); by_rank != 0: [k*n + r], else [k*n + gid]
 *   makespan[K], busy[K*d], transfer[K*d], peak[K*d] (int64), feasible[K]
 *   order[K*n]      optional (NULL): gids in dispatch order (ready-queue pops)
 *   err[1]          optional (NULL): set to 1 if any device id >= d (that
 *                   placement's outputs are NaN / 0) */
int dp_simulate_batch(const dp_graph *g, int32_t K, const uint8_t *placement, int32_t by_rank,
                      double *makespan, double *busy, double *transfer, int64_t *peak,
                      uint8_t *feasible, int32_t *order, uint8_t *err, void *stream);

/* ----------------------------------------------------------------- policy */

/* Create the device policy engine for one grouped graph's features and the
 * policy hyper-parameters (pkg/policy.py:45-114, 120-146).  Uploads the
 * structural features once (GroupFeatures.from_grouped, pkg/policy.py:97-114):
 *   h_type_off[T+1], h_type_idx[...]  type-vocab indices per decode step
 *                                      (sorted type names, with multiplicity)
 *   h_shape[T*shape_slots], h_adj[T*adj_slots]
 * and allocates activations for up to k_max samples.  hidden must be 64,
 * 1 <= n_dev <= 32, 1 <= dev_dim <= 32. */
int dp_policy_create(int32_t T, int32_t n_dev, int32_t hidden, int32_t dev_dim, int32_t type_dim,
                     int32_t shape_slots, int32_t adj_slots, int32_t vocab_rows, const int32_t *h_type_off,
                     const int32_t *h_type_idx, const double *h_shape, const double *h_adj, int32_t k_max,
                     dp_policy **out);
void dp_policy_destroy(dp_policy *p);
/* Length of the flat parameter vector (PolicyParams.flat_size, pkg/policy.py:164-166). */
int64_t dp_policy_num_params(const dp_policy *p);

/* Encoder for a parameter snapshot `params` (flat f64 [P], canonical _FIELDS
 * order, pkg/policy.py:41-42): input assembly, LSTM encoder over the T
 * groups in topo order and the decoder input table (pkg/policy.py:256-287).
 * Runs once per snapshot; all decode calls reuse it. */
int dp_policy_encode(dp_policy *p, const double *params, void *stream);

/* Debug instrumentation: enable/disable per-phase cycle counters in the
 * decoder (block 0) and the encoder and read+reset the 16 sums into h_out[16]
 * (may be NULL). */
int dp_debug_phase_clocks(int32_t enable, int64_t *h_out);

/* Debug instrumentation: the decoder's per-warp phase-end arrival cycles
 * (block 0, from each phase's start, summed over steps; phase clocks must be
 * enabled) into h_out[8 * 3], warp-major; read and reset. */
int dp_debug_warp_clocks(int64_t *h_out);

/* Debug instrumentation: LSTM-backward phase clocks (block 0) into h_out[8]. */
int dp_debug_lstm_clocks(int32_t enable, int64_t *h_out);

/* Debug instrumentation: attention-backward phase clocks (block 0, summed over
 * its chunks) into h_out[8]: wait + barrier, DA + ds, barrier, dq, dE + dA,
 * partial stores, barrier, tile prologue/epilogue. */
int dp_debug_att_clocks(int32_t enable, int64_t *h_out);

/* Accuracy check of the branch-free fp64 transcendentals (fastmath.cuh) the
 * recurrent kernels use, against the CUDA libm over n arguments per function:
 * h_max_ulps[5] = max ulp distance of {sigmoid, tanh, exp, expm1, division}. */
int dp_debug_fastmath_error(int64_t n, uint64_t *h_max_ulps);

/* Decoder variant override (tests / measurement): 0 = automatic plan,
 * 1 = force the speculative next-step cell (idle warps evaluate the LSTM
 * cell for every possible choice during the draw), 2 = forbid it, 4 = the
 * FAST decoder with its gate mat-vec h W_h on tcgen05 (int8 digit planes of
 * W_h resident in TMEM; measured slower at C3, so opt-in). */
int dp_debug_decoder_variant(int32_t mode);

/* Encoder recurrence override (tests / measurement): 0 = one CTA (default),
 * 1 = a 4-CTA cluster, each CTA a quarter of the gate columns, h exchanged
 * every step through distributed shared memory (st.async completing an
 * mbarrier transaction count; measured slower, so opt-in). */
int dp_debug_encoder_variant(int32_t mode);

/* Debug (tests): the decoder plan for a batch of K samples on this engine:
 * out[6] = {samples per CTA, kernel sample slots, tensor-core gates (0/1),
 * shared-memory bytes, speculative cell (0/1), operands in shared memory (0/1)}. */
int dp_debug_decoder_plan(const dp_policy *p, int32_t K, int32_t *out);

/* Debug (tests): free the optional backward stores of an engine so small
 * batches run the code paths a C5-sized batch takes.  mask bit 0 = attention
 * numerators (the attention backward recomputes the scores), bit 1 = per-tile
 * attention partials (backward_rows is a no-op; backward_grads runs the fused
 * backward). */
int dp_debug_policy_drop_stores(dp_policy *p, int32_t mask);

/* Graph ingestion on the device: per-group features and the
 * deduplicated group-edge CSR of a grouped op graph (reference GroupedGraph,
 * pkg/graph.py:183-238, and GroupFeatures.from_grouped, pkg/policy.py:97-114),
 * all indexed by GROUP ID (the caller orders rows by its topological rank).
 *   h_op_group[n_ops]     group id of each op
 *   h_op_key[n_ops]       rank of the op's type name among the sorted names
 *   h_key_to_index[n_keys] EmbeddingSpec row of each key (unknown -> last row)
 *   h_op_elems[n_ops]     output element count (0 for a scalar output)
 *   h_e_src/dst/bytes[n_edges]  op edges
 * Outputs (host): type_off[G+1] / type_idx[n_ops] (multiset in key order),
 * shape[G*shape_slots] (log1p of the largest counts, descending), adj[G*adj_slots]
 * (multi-hot of in + out neighbour groups mod adj_slots), ge_off[G+1] /
 * ge_dst[<= n_edges] / ge_bytes (out-edges to other groups, by destination,
 * summed bytes), out_bytes[G] (all member out-edges incl. intra-group).
 * Limits: <= 1024 type names, <= 2048 members / leaving edges per group. */
int dp_group_features(int32_t n_ops, int32_t n_groups, const int32_t *h_op_group, const int32_t *h_op_key,
                      int32_t n_keys, const int32_t *h_key_to_index, const int64_t *h_op_elems, int32_t n_edges,
                      const int32_t *h_e_src, const int32_t *h_e_dst, const int64_t *h_e_bytes, int32_t shape_slots,
                      int32_t adj_slots, int32_t *h_type_off, int32_t *h_type_idx, double *h_shape, double *h_adj,
                      int32_t *h_ge_off, int32_t *h_ge_dst, int64_t *h_ge_bytes, int64_t *h_out_bytes);

/* Debug (tests, A/B timing): mode 1 runs the fp64 DMMA / SIMT kernels where a
 * tcgen05 tensor-core path exists (the decoder weight gradient); 0 (default)
 * uses the tensor cores for the decoder weight gradient; 2 = the same with the
 * accumulators drained every 3 steps (the long-batch path, at small sizes);
 * 3-5 = timing ablations of that kernel (results invalid); 6 = additionally
 * the attention backward's digit-plane tcgen05 kernel (att_tc.cu), which
 * measures slower than the fp64 DMMA kernel at C3 and is not the default. */
int dp_debug_tensor_core(int32_t mode);

/* Copy the assembled encoder inputs of the last encode (embed_groups(),
 * pkg/policy.py:266-268) into out[T*input_dim] (device). */
int dp_policy_read_inputs(const dp_policy *p, double *out, void *stream);

/* Decode K samples from the encoded snapshot — forward_sample() /
 * log_prob_of() / step_distributions() (pkg/policy.py:288-340).
 *   h_pcg[4]      numpy PCG64 state (state_hi, state_lo, inc_hi, inc_lo) of the
 *                 caller's Generator; sample k, step t consumes draw
 *                 draw_base + (draw_counter ? *draw_counter * draws_per_count : 0)
 *                 + (k_offset + k)*T + t, i.e. exactly the draws K sequential
 *                 forward_sample calls would consume.
 *   forced[K*T]   optional (device): teacher-forced choices by rank instead of
 *                 sampling (then h_pcg may be NULL)
 *   choice_out[K*T] optional (device): sampled device per rank
 *   logp[K]       (device) log-probability of each placement
 *   probs_out[K*T*n_dev] optional (device): per-step distributions
 *   margin[K]     optional (device, sampling only): per sample, the minimum over
 *                 its T draws of min_{j < n_dev-1} |r - cdf_j| — how far each
 *                 uniform was from flipping the searchsorted choice
 *                 (pkg/policy.py:320-323).  +inf when n_dev == 1.
 * The activations of the last decode stay in the engine (the forward cache
 * used by dp_policy_backward). */
int dp_policy_decode(dp_policy *p, const double *params, int32_t K, int64_t k_offset, const uint64_t *h_pcg,
                     uint64_t draw_base, const int64_t *draw_counter, int64_t draws_per_count,
                     const uint8_t *forced, uint8_t *choice_out, double *logp, double *probs_out, double *margin,
                     void *stream);

/* grad[P] = sum_k adv[k] * d log p(placement_k) / d params over the samples of
 * the last decode call (K must match) — grad_log_prob() weighted and summed as
 * in reinforce_update() (pkg/policy.py:351-409, pkg/trainer.py:147-151). */
int dp_policy_backward(dp_policy *p, const double *params, int32_t K, const double *adv, double *grad,
                       void *stream);

/* The same gradient in two halves so the first overlaps the simulator:
 * _rows: the advantage-independent per-(sample, step) work (everything is
 *        linear in adv, so it runs with adv := 1) — needs no scores;
 * _grads: the advantage-weighted cross-sample sums.  Falls back to the fused
 *        pass when _rows did not run for this decode (or the alpha store would
 *        exceed the memory budget).  _rows and _grads may run on different
 *        streams: _grads orders itself after _rows with events recorded by
 *        _rows (its attention sums start when the attention backward is done,
 *        the rest when the whole rows pass is). */
int dp_policy_backward_rows(dp_policy *p, const double *params, int32_t K, void *stream);
int dp_policy_backward_grads(dp_policy *p, const double *params, int32_t K, const double *adv, double *grad,
                             void *stream);

/* ---------------------------------------------------------------- trainer */

/* Device-resident controller state (one per controller); zero-initialise,
 * then set baseline = failing signal and best_r = +inf (pkg/trainer.py:263-267). */
typedef struct {
    double baseline;      /* BaselineState.value */
    double baseline_prev; /* B used for this update's advantages */
    double best_r;        /* best feasible reward so far (+inf if none) */
    int64_t update;       /* controller-local update index */
    int64_t adam_t;       /* ParameterStore._t */
    int64_t version;      /* ParameterStore.version */
    int64_t rejected;     /* ParameterStore.rejected */
    int64_t n_used;
    int64_t n_feasible;
    int64_t best_update;
    int64_t best_k;
    int64_t error;        /* 1: a feasible measurement was not positive/finite */
} dp_train_state;

/* Simulator variant override (tests / measurement): 0 = automatic, 1 = one
 * warp per placement, 2 = one thread per placement. */
int dp_debug_sim_variant(int32_t mode);

/* Batched search baselines on K-sim (pkg/baselines.py:227-273).
 * dp_enumerate_placements: out[count*n] (by gid) = placements start..start+
 *   count-1 of itertools.product(range(d), repeat=n) (last group fastest).
 * dp_argmin_feasible: folds the first minimal feasible makespan of a batch
 *   (global index base_index + k) into (*best_val, *best_idx) with a strict <
 *   (earlier batches keep ties); *best_idx = -1 initially. */
int dp_enumerate_placements(int32_t n, int32_t d, uint64_t start, int32_t count, uint8_t *out, void *stream);
int dp_argmin_feasible(int32_t K, const double *makespan, const uint8_t *feasible, int64_t base_index,
                       double *best_val, int64_t *best_idx, void *stream);

/* Rewards, best-so-far, success-only filter, baseline and advantages for one
 * update (pkg/trainer.py:66-72, 83-84, 138-154, 281-304), on device:
 *   makespan[K], feasible[K]: all K samples of the update
 *   choice: placement rows by rank; the best sample k's row is
 *           choice[(k / choice_div) * T ..] — choice_div = 1: all K rows;
 *           choice_div = K_local: one candidate row per rank (the K-sharded
 *           exchange gathers only each rank's local best, dp_exchange_pack)
 *   adv[K_local] (out): (R_k - B) for used samples k_offset.. else 0
 *   best_choice[T] (out): updated when the best reward improves
 *   log_rows[log_cap*8] (out): row `update` = (update, controller, version,
 *   mean_R, baseline, best_R, n_feasible, n_used); version is filled by
 *   dp_adam_apply. */
/* Sampling certificate (reference draw pkg/policy.py:320-323):
 * margin_min[0] = min(margin_min[0], min_k margin[k]) and n_below[0] += #{k :
 * margin[k] < tol} over the per-sample margins of one dp_policy_decode. */
int dp_margin_accumulate(int32_t K, const double *margin, double tol, double *margin_min, int64_t *n_below,
                         void *stream);

int dp_reinforce_epilogue(int32_t K, int32_t T, const double *makespan, const uint8_t *feasible,
                          const uint8_t *choice, int32_t choice_div, double failing, double decay,
                          int64_t success_only_after,
                          int64_t k_offset, int32_t K_local, dp_train_state *state, double *adv,
                          uint8_t *best_choice, double *log_rows, int64_t log_cap, int32_t controller_id,
                          void *stream);

/* measure() with lognormal noise (pkg/simulator.py:205-223, pkg/trainer.py:
 * 244-253, 277): for every feasible k, makespan[k] <- np.mean(makespan[k] *
 * factors[update][k][0..n_factors)) in numpy's pairwise order, update =
 * state->update.  factors = exp(sigma * default_rng(seed_k).standard_normal(
 * steps))[1:] per sample, seeds from the controller's noise stream (host).
 * K-sharded: makespan/feasible hold samples k_offset..k_offset+K-1 of K_total
 * (factor rows [update][k_offset + k]).
 * Sets state->error = 2 if update >= n_updates. */
int dp_apply_measurement_noise(int32_t K, int64_t k_offset, int32_t K_total, double *makespan,
                               const uint8_t *feasible, const double *factors, int64_t n_updates,
                               int32_t n_factors, dp_train_state *state, void *stream);

/* K-sharded exchange buffers.  A rank's record is
 * dp_exchange_record_bytes(K_local, T) bytes: makespan f64[K_local] |
 * feasible u8[K_local] | its best candidate's placement row u8[T] (by rank;
 * the first feasible sample with the smallest reward sqrt(makespan), the rule
 * of pkg/trainer.py:284-287 restricted to the shard) — padded to 16 bytes.
 * pack: local scores + choice[K_local*T] -> record.  unpack: the all-gathered
 * records [nranks] -> makespan[K], feasible[K], rows[nranks*T] (the epilogue's
 * choice with choice_div = K_local). */
int64_t dp_exchange_record_bytes(int32_t K_local, int32_t T);
int dp_exchange_pack(int32_t K_local, int32_t T, const double *makespan, const uint8_t *feasible,
                     const uint8_t *choice, uint8_t *record, void *stream);
int dp_exchange_unpack(int32_t nranks, int32_t K_local, int32_t T, const uint8_t *records, double *makespan,
                       uint8_t *feasible, uint8_t *rows, void *stream);

/* NCCL (dlopen'ed libnccl.so.2) for the K-sharded step; DP_ECOMM on failure.
 * One process per GPU: dp_comm_unique_id on rank 0, broadcast the 128 bytes,
 * dp_comm_init_rank on every rank (current CUDA device).  One process for all
 * GPUs: dp_comm_init_all (one communicator per device).  With several
 * communicators in one thread, wrap the per-device calls in
 * dp_comm_group_start/end.  All collectives enqueue on `stream` and are CUDA
 * graph capturable. */
typedef struct dp_comm dp_comm;
int dp_comm_version(int32_t *version);
int dp_comm_unique_id(uint8_t *id_out /* [128] */);
int dp_comm_init_rank(int32_t nranks, const uint8_t *id /* [128] */, int32_t rank, dp_comm **out);
int dp_comm_init_all(int32_t ndev, const int32_t *devices, dp_comm **out /* [ndev] */);
void dp_comm_destroy(dp_comm *c);
int dp_comm_group_start(void);
int dp_comm_group_end(void);
int dp_comm_all_gather(dp_comm *c, const void *send, void *recv, int64_t bytes_per_rank, void *stream);
int dp_comm_all_reduce_f64(dp_comm *c, double *buf, int64_t count, int32_t op_min, void *stream);

/* ParameterStore.apply (pkg/trainer.py:113-131): grad is the advantage-weighted
 * SUM from dp_policy_backward; it is divided by n_used here.  Skips the step
 * when n_used == 0 (reinforce_update returned None), rejects non-finite
 * gradients (rejected++), else Adam with bias_corr[2*(t-1)+{0,1}] =
 * 1-b1^t, 1-b2^t (host-computed Python floats) and version++.  Then advances
 * state->update.  flag: device int32 scratch, zero-initialised.
 * store_state: the shared ParameterStore's counters (adam_t, version,
 * rejected) when several controllers share one store (pkg/trainer.py:365-378);
 * NULL = state (single controller).  A step beyond t_cap (the bias-correction
 * table's length) sets state->error = 3 and leaves everything unchanged. */
int dp_adam_apply(int64_t P, double *params, double *m, double *v, const double *grad, const double *bias_corr,
                  int64_t t_cap, double lr, double b1, double b2, double eps, dp_train_state *state,
                  dp_train_state *store_state, int32_t *flag, double *log_rows, int64_t log_cap, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* DEVPLACE_B200_H */
