// Shared helpers for the devplace_b200 sm_100a kernels.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string>

#include "../../include/devplace_b200.h"

namespace dp {

void set_error(const std::string &msg);
// Opt a kernel into > 48 KB dynamic shared memory on the current device (cached).
cudaError_t allow_big_smem(const void *func, size_t bytes);

#define DP_CUDA_TRY(expr)                                                                  \
    do {                                                                                   \
        cudaError_t e_ = (expr);                                                           \
        if (e_ != cudaSuccess) {                                                           \
            ::dp::set_error(std::string(#expr) + ": " + cudaGetErrorString(e_));           \
            return DP_ECUDA;                                                               \
        }                                                                                  \
    } while (0)

// Entry-point prologue: clear a stale runtime error left by an unrelated call
// (e.g. a cudaFree from a destructor) so it is not misattributed.  Sticky
// (context-corrupting) errors persist and still surface.
#define DP_ENTRY() (void)cudaGetLastError()

#define DP_REQUIRE(cond, msg)                                                            \
    do {                                                                                   \
        if (!(cond)) {                                                                     \
            ::dp::set_error(msg);                                                          \
            return DP_EINVAL;                                                              \
        }                                                                                  \
    } while (0)

// Every kernel launch goes through DP_LAUNCH_CHECK, which also counts it
// (dp_launch_count(): evidence of how many of our kernels a step enqueues).
void count_launch();

#define DP_LAUNCH_CHECK()                                                                  \
    do {                                                                                   \
        ::dp::count_launch();                                                              \
        cudaError_t e_ = cudaGetLastError();                                               \
        if (e_ != cudaSuccess) {                                                           \
            ::dp::set_error(std::string("kernel launch at ") + __FILE__ + ":" +            \
                            std::to_string(__LINE__) + ": " + cudaGetErrorString(e_));     \
            return DP_ECUDA;                                                               \
        }                                                                                  \
    } while (0)

constexpr int kNumSMs = 148;

static inline int ceil_div(long long a, long long b) { return (int)((a + b - 1) / b); }

}  // namespace dp

// Device graph (see dp_graph_create): everything indexed by topo rank.
struct dp_graph {
    int32_t n, d, e;
    double *cost;        // [n]
    double *dur;         // [n*d] cost[r] / rate[dev], host-computed (IEEE, same as Python)
    int32_t *indeg;      // [n]
    int32_t *out_off;    // [n+1]
    int32_t *out_dst;    // [e]
    double *out_bytes;   // [e] exact for < 2^53, else rounded like Python float(int)
    int64_t *resident;   // [n]
    int32_t *gid;        // [n] gid of rank
    int32_t *rank;       // [n] rank of gid
    double *rate;        // [d]
    double *bw;          // [d*d]
    int64_t *mem;        // [d]
    int32_t max_indeg;
    size_t sim_smem_per_placement;
    // shared-memory image of the graph (dur | out_bytes | bw | out_off | dst u16 |
    // gid u16 | indeg u16, 16-byte padded) staged with one TMA bulk copy
    unsigned char *image;
    size_t image_bytes;
};
