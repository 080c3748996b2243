// Graph ingestion on the device: per-group policy features
// and the deduplicated group-edge CSR for paper-scale op graphs.
//
// Reference: GroupedGraph construction (/root/reference/pkg/src/devplace/
// graph.py:183-238: out_bytes over all member out-edges, cross-group edges
// deduplicated with summed bytes, sorted by (src, dst)) and
// GroupFeatures.from_grouped (policy.py:97-114: type indices with
// multiplicity in sorted type-name order, log1p of member output element
// counts sorted descending into shape_slots, multi-hot of in + out neighbour
// group ids mod adjacency_slots).  Everything is by group id; the host orders
// the rows by the Kahn topological rank (graph.py:252-266) it computes from
// the returned CSR.
//
// Integer work (counts, scans, scatters, per-group sorts): one CTA per group
// for the per-group pieces, grid-stride kernels for the op/edge passes.

#include <math.h>

#include <algorithm>
#include <climits>
#include <vector>

#include "common.cuh"

namespace dp {
namespace {

constexpr int kFt = 256;        // threads per CTA
constexpr int kMaxKeys = 1024;    // distinct op types
constexpr int kMaxBucket = 2048;  // members / leaving edges of one group (shared-memory sorts)
constexpr int kMaxShape = 64;

__global__ void ft_count(int n_ops, const int32_t *__restrict__ op_group, int n_edges, const int32_t *__restrict__ e_src,
                         const int32_t *__restrict__ e_dst, const int64_t *__restrict__ e_bytes, int32_t *cnt_mem,
                         int32_t *cnt_cross, unsigned long long *out_bytes) {
    const int stride = gridDim.x * blockDim.x;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n_ops; i += stride) atomicAdd(cnt_mem + op_group[i], 1);
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n_edges; e += stride) {
        const int gs = op_group[e_src[e]], gd = op_group[e_dst[e]];
        atomicAdd(out_bytes + gs, (unsigned long long)e_bytes[e]);
        if (gs != gd) atomicAdd(cnt_cross + gs, 1);
    }
}

// exclusive scan of n counts -> off[n + 1] (one CTA; n up to a few 1e5)
__global__ void ft_scan(int n, const int32_t *__restrict__ cnt, int32_t *__restrict__ off) {
    __shared__ int32_t part[kFt];
    const int per = (n + kFt - 1) / kFt;
    const int b = threadIdx.x * per, e = min(n, b + per);
    int32_t s = 0;
    for (int i = b; i < e; i++) s += cnt[i];
    part[threadIdx.x] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        int32_t run = 0;
        for (int i = 0; i < kFt; i++) {
            const int32_t v = part[i];
            part[i] = run;
            run += v;
        }
        off[n] = run;
    }
    __syncthreads();
    int32_t run = part[threadIdx.x];
    for (int i = b; i < e; i++) {
        off[i] = run;
        run += cnt[i];
    }
}

__global__ void ft_scatter(int n_ops, const int32_t *__restrict__ op_group, int n_edges,
                           const int32_t *__restrict__ e_src, const int32_t *__restrict__ e_dst,
                           const int64_t *__restrict__ e_bytes, const int32_t *__restrict__ mem_off,
                           const int32_t *__restrict__ cross_off, int32_t *fill_mem, int32_t *fill_cross,
                           int32_t *members, int32_t *cross_dst, int64_t *cross_bytes) {
    const int stride = gridDim.x * blockDim.x;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n_ops; i += stride) {
        const int g = op_group[i];
        members[mem_off[g] + atomicAdd(fill_mem + g, 1)] = i;
    }
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n_edges; e += stride) {
        const int gs = op_group[e_src[e]], gd = op_group[e_dst[e]];
        if (gs == gd) continue;
        const int slot = cross_off[gs] + atomicAdd(fill_cross + gs, 1);
        cross_dst[slot] = gd;
        cross_bytes[slot] = e_bytes[e];
    }
}

// descending bitonic sort of n (power of two) keys in shared memory
__device__ void bitonic_desc(long long *v, int n, int tid) {
    for (int k = 2; k <= n; k <<= 1)
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = tid; i < n; i += kFt) {
                const int p = i ^ j;
                if (p > i) {
                    const bool down = (i & k) == 0;
                    if ((v[i] < v[p]) == down) {
                        const long long t = v[i];
                        v[i] = v[p];
                        v[p] = t;
                    }
                }
            }
            __syncthreads();
        }
}

// one CTA per group: type multiset (key order), top shape_slots output element
// counts, and the group's deduplicated out-edges sorted by destination group
__global__ void __launch_bounds__(kFt) ft_group(int n_keys, const int32_t *__restrict__ op_key,
                                                const int32_t *__restrict__ key_to_index,
                                                const int64_t *__restrict__ op_elems,
                                                const int32_t *__restrict__ mem_off,
                                                const int32_t *__restrict__ members, const int32_t *__restrict__ cross_off,
                                                int32_t *__restrict__ cross_dst, int64_t *__restrict__ cross_bytes,
                                                int shape_slots, int32_t *__restrict__ type_idx,
                                                double *__restrict__ shape, int32_t *__restrict__ n_dedup) {
    __shared__ int32_t hist[kMaxKeys];
    __shared__ int32_t hoff[kMaxKeys];
    __shared__ int32_t sdst[kMaxBucket];
    __shared__ long long sbytes[kMaxBucket];
    const int g = blockIdx.x, tid = threadIdx.x;
    const int m0 = mem_off[g], m1 = mem_off[g + 1];
    // ---- type multiset in key (sorted type-name) order
    for (int k = tid; k < n_keys; k += kFt) hist[k] = 0;
    __syncthreads();
    for (int i = m0 + tid; i < m1; i += kFt) atomicAdd(hist + op_key[members[i]], 1);
    __syncthreads();
    if (tid == 0) {
        int32_t run = 0;
        for (int k = 0; k < n_keys; k++) {
            hoff[k] = run;
            run += hist[k];
        }
    }
    __syncthreads();
    for (int k = tid; k < n_keys; k += kFt) {
        const int32_t ix = key_to_index[k];
        for (int j = 0; j < hist[k]; j++) type_idx[m0 + hoff[k] + j] = ix;
    }
    // ---- shape block: the shape_slots largest positive element counts, descending
    {
        const int nm = m1 - m0;
        int np2 = 1;
        while (np2 < nm) np2 <<= 1;
        for (int i = tid; i < np2; i += kFt) sbytes[i] = i < nm ? op_elems[members[m0 + i]] : 0;  // non-positive sort last
        __syncthreads();
        bitonic_desc(sbytes, np2, tid);
        double *srow = shape + (size_t)g * shape_slots;
        for (int j = tid; j < shape_slots; j += kFt) srow[j] = j < nm && sbytes[j] > 0 ? log1p((double)sbytes[j]) : 0.0;
        __syncthreads();
    }
    // ---- out-edges to other groups: sort by destination, merge duplicates
    const int c0 = cross_off[g], nc = cross_off[g + 1] - c0;
    for (int i = tid; i < nc; i += kFt) {
        sdst[i] = cross_dst[c0 + i];
        sbytes[i] = cross_bytes[c0 + i];
    }
    int np2 = 1;
    while (np2 < nc) np2 <<= 1;
    for (int i = nc + tid; i < np2; i += kFt) sdst[i] = INT_MAX, sbytes[i] = 0;
    __syncthreads();
    // bitonic sort on (dst); equal keys are merged below, so stability is irrelevant
    for (int k = 2; k <= np2; k <<= 1)
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = tid; i < np2; i += kFt) {
                const int p = i ^ j;
                if (p > i) {
                    const bool up = (i & k) == 0;
                    if ((sdst[i] > sdst[p]) == up) {
                        const int32_t td = sdst[i];
                        sdst[i] = sdst[p];
                        sdst[p] = td;
                        const long long tb = sbytes[i];
                        sbytes[i] = sbytes[p];
                        sbytes[p] = tb;
                    }
                }
            }
            __syncthreads();
        }
    if (tid == 0) {
        int w = 0;
        for (int i = 0; i < nc; i++) {
            if (w > 0 && sdst[i] == cross_dst[c0 + w - 1]) {
                cross_bytes[c0 + w - 1] += sbytes[i];
            } else {
                cross_dst[c0 + w] = sdst[i];
                cross_bytes[c0 + w] = sbytes[i];
                w++;
            }
        }
        n_dedup[g] = w;
    }
}

// compact the deduplicated rows; adjacency multi-hot of in + out neighbours
__global__ void ft_compact(int n_groups, const int32_t *__restrict__ cross_off, const int32_t *__restrict__ cross_dst,
                           const int64_t *__restrict__ cross_bytes, const int32_t *__restrict__ ge_off,
                           int32_t *__restrict__ ge_dst, int64_t *__restrict__ ge_bytes, int adj_slots,
                           double *__restrict__ adj) {
    const int g = blockIdx.x;
    const int o = ge_off[g], n = ge_off[g + 1] - o, c0 = cross_off[g];
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const int d = cross_dst[c0 + i];
        ge_dst[o + i] = d;
        ge_bytes[o + i] = cross_bytes[c0 + i];
        adj[(size_t)g * adj_slots + d % adj_slots] = 1.0;  // out-neighbour
        adj[(size_t)d * adj_slots + g % adj_slots] = 1.0;  // g is an in-neighbour of d
    }
}

}  // namespace
}  // namespace dp

using namespace dp;

extern "C" int dp_group_features(int32_t n_ops, int32_t n_groups, const int32_t *h_op_group, const int32_t *h_op_key,
                                 int32_t n_keys, const int32_t *h_key_to_index, const int64_t *h_op_elems,
                                 int32_t n_edges, const int32_t *h_e_src, const int32_t *h_e_dst,
                                 const int64_t *h_e_bytes, int32_t shape_slots, int32_t adj_slots,
                                 int32_t *h_type_off, int32_t *h_type_idx, double *h_shape, double *h_adj,
                                 int32_t *h_ge_off, int32_t *h_ge_dst, int64_t *h_ge_bytes, int64_t *h_out_bytes) {
    DP_ENTRY();
    DP_REQUIRE(n_ops >= 1 && n_groups >= 1 && n_edges >= 0, "dp_group_features: empty graph");
    DP_REQUIRE(n_keys >= 1 && n_keys <= kMaxKeys, "dp_group_features: need 1 <= distinct op types <= 1024");
    DP_REQUIRE(shape_slots >= 1 && shape_slots <= kMaxShape && adj_slots >= 1,
               "dp_group_features: need 1 <= shape_slots <= 64 and adjacency_slots >= 1");
    for (int i = 0; i < n_ops; i++) {
        DP_REQUIRE(h_op_group[i] >= 0 && h_op_group[i] < n_groups, "dp_group_features: op group out of range");
        DP_REQUIRE(h_op_key[i] >= 0 && h_op_key[i] < n_keys, "dp_group_features: op type key out of range");
    }
    for (int e = 0; e < n_edges; e++)
        DP_REQUIRE(h_e_src[e] >= 0 && h_e_src[e] < n_ops && h_e_dst[e] >= 0 && h_e_dst[e] < n_ops,
                   "dp_group_features: dangling edge endpoint");
    // device buffers (one allocation, carved)
    const size_t G = n_groups, N = n_ops, E = n_edges > 0 ? n_edges : 1;
    size_t bytes = 0;
    auto take = [&](size_t nb) {
        const size_t o = bytes;
        bytes += (nb + 255) & ~(size_t)255;
        return o;
    };
    const size_t o_group = take(4 * N), o_key = take(4 * N), o_k2i = take(4 * (size_t)n_keys), o_elems = take(8 * N),
                 o_src = take(4 * E), o_dst = take(4 * E), o_eb = take(8 * E), o_cnt_mem = take(4 * G),
                 o_cnt_cross = take(4 * G), o_outb = take(8 * G), o_mem_off = take(4 * (G + 1)),
                 o_cross_off = take(4 * (G + 1)), o_fill_mem = take(4 * G), o_fill_cross = take(4 * G),
                 o_members = take(4 * N), o_cdst = take(4 * E), o_cbytes = take(8 * E), o_tidx = take(4 * N),
                 o_shape = take(8 * G * shape_slots), o_adj = take(8 * G * adj_slots), o_ndd = take(4 * G),
                 o_ge_off = take(4 * (G + 1)), o_ge_dst = take(4 * E), o_ge_bytes = take(8 * E);
    uint8_t *d = nullptr;
    DP_CUDA_TRY(cudaMalloc(&d, bytes));
    auto P = [&](size_t o) { return (void *)(d + o); };
    int rc = DP_OK;
    do {
        cudaStream_t st = 0;
#define FT_TRY(x)                         \
    if ((x) != cudaSuccess) {             \
        ::dp::set_error(cudaGetErrorString(cudaGetLastError())); \
        rc = DP_ECUDA;                    \
        break;                            \
    }
        FT_TRY(cudaMemsetAsync(d, 0, bytes, st));
        FT_TRY(cudaMemcpyAsync(P(o_group), h_op_group, 4 * N, cudaMemcpyHostToDevice, st));
        FT_TRY(cudaMemcpyAsync(P(o_key), h_op_key, 4 * N, cudaMemcpyHostToDevice, st));
        FT_TRY(cudaMemcpyAsync(P(o_k2i), h_key_to_index, 4 * (size_t)n_keys, cudaMemcpyHostToDevice, st));
        FT_TRY(cudaMemcpyAsync(P(o_elems), h_op_elems, 8 * N, cudaMemcpyHostToDevice, st));
        if (n_edges) {
            FT_TRY(cudaMemcpyAsync(P(o_src), h_e_src, 4 * (size_t)n_edges, cudaMemcpyHostToDevice, st));
            FT_TRY(cudaMemcpyAsync(P(o_dst), h_e_dst, 4 * (size_t)n_edges, cudaMemcpyHostToDevice, st));
            FT_TRY(cudaMemcpyAsync(P(o_eb), h_e_bytes, 8 * (size_t)n_edges, cudaMemcpyHostToDevice, st));
        }
        const int grid = 2 * kNumSMs;
        ft_count<<<grid, kFt, 0, st>>>(n_ops, (int32_t *)P(o_group), n_edges, (int32_t *)P(o_src), (int32_t *)P(o_dst),
                                       (int64_t *)P(o_eb), (int32_t *)P(o_cnt_mem), (int32_t *)P(o_cnt_cross),
                                       (unsigned long long *)P(o_outb));
        ft_scan<<<1, kFt, 0, st>>>(n_groups, (int32_t *)P(o_cnt_mem), (int32_t *)P(o_mem_off));
        ft_scan<<<1, kFt, 0, st>>>(n_groups, (int32_t *)P(o_cnt_cross), (int32_t *)P(o_cross_off));
        ft_scatter<<<grid, kFt, 0, st>>>(n_ops, (int32_t *)P(o_group), n_edges, (int32_t *)P(o_src),
                                         (int32_t *)P(o_dst), (int64_t *)P(o_eb), (int32_t *)P(o_mem_off),
                                         (int32_t *)P(o_cross_off), (int32_t *)P(o_fill_mem),
                                         (int32_t *)P(o_fill_cross), (int32_t *)P(o_members), (int32_t *)P(o_cdst),
                                         (int64_t *)P(o_cbytes));
        FT_TRY(cudaGetLastError());
        // bucket-size limit of the in-CTA sort
        std::vector<int32_t> cross_off(G + 1);
        FT_TRY(cudaMemcpyAsync(cross_off.data(), P(o_cross_off), 4 * (G + 1), cudaMemcpyDeviceToHost, st));
        FT_TRY(cudaStreamSynchronize(st));
        std::vector<int32_t> mem_off(G + 1);
        FT_TRY(cudaMemcpy(mem_off.data(), P(o_mem_off), 4 * (G + 1), cudaMemcpyDeviceToHost));
        int big = 0;
        for (size_t g = 0; g < G; g++)
            big = std::max(big, std::max(cross_off[g + 1] - cross_off[g], mem_off[g + 1] - mem_off[g]));
        if (big > kMaxBucket) {
            ::dp::set_error("dp_group_features: a group has more than 2048 members or leaving edges");
            rc = DP_EINVAL;
            break;
        }
        ft_group<<<n_groups, kFt, 0, st>>>(n_keys, (int32_t *)P(o_key), (int32_t *)P(o_k2i), (int64_t *)P(o_elems),
                                           (int32_t *)P(o_mem_off), (int32_t *)P(o_members), (int32_t *)P(o_cross_off),
                                           (int32_t *)P(o_cdst), (int64_t *)P(o_cbytes), shape_slots,
                                           (int32_t *)P(o_tidx), (double *)P(o_shape), (int32_t *)P(o_ndd));
        ft_scan<<<1, kFt, 0, st>>>(n_groups, (int32_t *)P(o_ndd), (int32_t *)P(o_ge_off));
        ft_compact<<<n_groups, 128, 0, st>>>(n_groups, (int32_t *)P(o_cross_off), (int32_t *)P(o_cdst),
                                             (int64_t *)P(o_cbytes), (int32_t *)P(o_ge_off), (int32_t *)P(o_ge_dst),
                                             (int64_t *)P(o_ge_bytes), adj_slots, (double *)P(o_adj));
        FT_TRY(cudaGetLastError());
        FT_TRY(cudaMemcpyAsync(h_type_off, P(o_mem_off), 4 * (G + 1), cudaMemcpyDeviceToHost, st));
        FT_TRY(cudaMemcpyAsync(h_type_idx, P(o_tidx), 4 * N, cudaMemcpyDeviceToHost, st));
        FT_TRY(cudaMemcpyAsync(h_shape, P(o_shape), 8 * G * shape_slots, cudaMemcpyDeviceToHost, st));
        FT_TRY(cudaMemcpyAsync(h_adj, P(o_adj), 8 * G * adj_slots, cudaMemcpyDeviceToHost, st));
        FT_TRY(cudaMemcpyAsync(h_ge_off, P(o_ge_off), 4 * (G + 1), cudaMemcpyDeviceToHost, st));
        FT_TRY(cudaMemcpyAsync(h_out_bytes, P(o_outb), 8 * G, cudaMemcpyDeviceToHost, st));
        FT_TRY(cudaStreamSynchronize(st));
        const int ne = h_ge_off[G];
        if (ne) {
            FT_TRY(cudaMemcpy(h_ge_dst, P(o_ge_dst), 4 * (size_t)ne, cudaMemcpyDeviceToHost));
            FT_TRY(cudaMemcpy(h_ge_bytes, P(o_ge_bytes), 8 * (size_t)ne, cudaMemcpyDeviceToHost));
        }
#undef FT_TRY
    } while (0);
    cudaFree(d);
    if (rc == DP_OK)
        for (int i = 0; i < 7; i++) ::dp::count_launch();  // count, 3 scans, scatter, group, compact
    return rc;
}
