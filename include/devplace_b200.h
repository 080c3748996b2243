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

typedef struct dp_graph dp_graph;
typedef struct dp_policy dp_policy;

/* Text of the last error raised on this thread ("" if none). */
const char *dp_last_error(void);

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
 * pkg/simulator.py:205-219).  One thread per placement, event-exact:
 * makespan/busy/transfer/peak/feasible and the dispatch order are bit-identical
 * to the reference.
 *   placement[K*n]  device ids (u8); by_rank != 0: [k*n + r], else [k*n + gid]
 *   makespan[K], busy[K*d], transfer[K*d], peak[K*d] (int64), feasible[K]
 *   order[K*n]      optional (NULL): gids in dispatch order (ready-queue pops)
 *   err[1]          optional (NULL): set to 1 if any device id >= d (that
 *                   placement's outputs are NaN / 0) */
int dp_simulate_batch(const dp_graph *g, int32_t K, const uint8_t *placement, int32_t by_rank,
                      double *makespan, double *busy, double *transfer, int64_t *peak,
                      uint8_t *feasible, int32_t *order, uint8_t *err, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* DEVPLACE_B200_H */
