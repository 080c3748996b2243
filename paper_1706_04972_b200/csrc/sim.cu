// K-sim: batched, event-exact placement simulator (sm_100a).
//
// Replaces simulate()/check_memory() of the reference cost model,
// /root/reference/pkg/src/devplace/simulator.py:93-194, for K placements per
// launch.  One thread owns one placement; its whole event state lives in
// shared memory (SoA, slot-interleaved so lanes at the same step touch
// consecutive words).  The graph (CSR by topo rank, durations, bytes) is
// read-only and shared by all placements through L1/L2.
//
// Exact restatement (verified bit-identical):
//   * per-edge ARRIVAL events collapse into one READY event per group, fired at
//     max(arrive) with key (t, kind=1, rank) — the key of the group's last
//     ARRIVAL in the reference heap;
//   * a device has at most one pending FINISH (t, kind=0, rank), so FINISH
//     events live in D slots instead of a heap;
//   * READY events are popped from a binary min-heap keyed (t, rank);
//   * a device's ready queue receives entries in READY-pop order, i.e. sorted
//     by (t, rank) except inside zero-duration cascades, so it is a sorted
//     array segment with tail insertion (usually O(1)).
// All fp64 operations (cost/rate, now+dur, bytes/bw, max, +=) are performed in
// the reference's order, so every output is bit-identical, including the
// dispatch order.  Compiled with --fmad=false (there are no mul-adds anyway).

#include "common.cuh"

namespace {

struct SimSlot {
    int S, s;
    __device__ __forceinline__ size_t at(int i) const { return (size_t)i * S + s; }
};

__device__ __forceinline__ bool key_less(double ta, int ra, double tb, int rb) {
    return ta < tb || (ta == tb && ra < rb);
}

// Bytes of the graph image staged in shared memory (GS=true).
__host__ __device__ inline size_t graph_smem_bytes(int n, int d, int e) {
    size_t b = 8 * ((size_t)n * d + e + (size_t)d * d) + 4 * (size_t)(n + 1) + 2 * ((size_t)e + 2 * n);
    return (b + 15) & ~(size_t)15;
}

// GS: stage the graph (durations, CSR, bytes, bandwidths) in shared memory
// once per CTA — every event's lookups become LDS instead of L2 round trips.
template <bool GS>
__global__ void __launch_bounds__(128) sim_kernel(dp_graph g, int K, const uint8_t *__restrict__ placement,
                                                  int by_rank, double *__restrict__ makespan,
                                                  double *__restrict__ busy_out, double *__restrict__ transfer_out,
                                                  int64_t *__restrict__ peak_out, uint8_t *__restrict__ feasible,
                                                  int32_t *__restrict__ order, uint8_t *__restrict__ err, int S) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int s = threadIdx.x;
    const int k = blockIdx.x * S + s;
    const int n = g.n, D = g.d;
    size_t gbytes = 0;
    const double *g_dur = g.dur, *g_bytes = g.out_bytes, *g_bw = g.bw;
    const int32_t *g_off = g.out_off;
    const int32_t *g_dst32 = g.out_dst, *g_gid32 = g.gid, *g_indeg32 = g.indeg;
    const uint16_t *g_dst16 = nullptr, *g_gid16 = nullptr, *g_indeg16 = nullptr;
    if (GS) {
        double *sdur = reinterpret_cast<double *>(smem);
        double *sbytes = sdur + (size_t)n * D;
        double *sbw = sbytes + g.e;
        int32_t *soff = reinterpret_cast<int32_t *>(sbw + D * D);
        uint16_t *sdst = reinterpret_cast<uint16_t *>(soff + n + 1);
        uint16_t *sgid = sdst + g.e;
        uint16_t *sind = sgid + n;
        for (int i = s; i < n * D; i += blockDim.x) sdur[i] = g.dur[i];
        for (int i = s; i < g.e; i += blockDim.x) {
            sbytes[i] = g.out_bytes[i];
            sdst[i] = (uint16_t)g.out_dst[i];
        }
        for (int i = s; i < D * D; i += blockDim.x) sbw[i] = g.bw[i];
        for (int i = s; i <= n; i += blockDim.x) soff[i] = g.out_off[i];
        for (int i = s; i < n; i += blockDim.x) {
            sgid[i] = (uint16_t)g.gid[i];
            sind[i] = (uint16_t)g.indeg[i];
        }
        __syncthreads();
        g_dur = sdur;
        g_bytes = sbytes;
        g_bw = sbw;
        g_off = soff;
        g_dst16 = sdst;
        g_gid16 = sgid;
        g_indeg16 = sind;
        gbytes = graph_smem_bytes(n, D, g.e);
    }
    auto dst_of = [&](int e) -> int { return GS ? (int)g_dst16[e] : g_dst32[e]; };
    auto gid_of = [&](int r) -> int { return GS ? (int)g_gid16[r] : g_gid32[r]; };
    auto indeg_of = [&](int r) -> int { return GS ? (int)g_indeg16[r] : g_indeg32[r]; };
    if (s >= S || k >= K) return;
    const SimSlot q{S, s};

    // ---- shared-memory carve-up (all arrays slot-interleaved: [i*S + s]) ----
    double *maxarr = reinterpret_cast<double *>(smem + gbytes);  // [n]  READY time (max arrival)
    double *fin_t = maxarr + (size_t)n * S;              // [D]  pending FINISH time per device
    double *link = fin_t + (size_t)D * S;                // [D*D] link_free
    double *busy = link + (size_t)D * D * S;             // [D]
    double *trans = busy + (size_t)D * S;                // [D]
    long long *peak = reinterpret_cast<long long *>(trans + (size_t)D * S);  // [D]
    int *fin_r = reinterpret_cast<int *>(peak + (size_t)D * S);              // [D] -1 = idle
    uint16_t *left = reinterpret_cast<uint16_t *>(fin_r + (size_t)D * S);    // [n] unfinished preds
    uint16_t *heap = left + (size_t)n * S;                                   // [n] READY heap (ranks)
    uint16_t *devq = heap + (size_t)n * S;                                   // [n] ready queues
    uint16_t *qhead = devq + (size_t)n * S;                                  // [D]
    uint16_t *qtail = qhead + (size_t)D * S;                                 // [D]
    uint8_t *pl = reinterpret_cast<uint8_t *>(qtail + (size_t)D * S);        // [n] device of rank

    // ---- placement load + validation (pkg/simulator.py:109-116) ----
    const uint8_t *src = placement + (size_t)k * n;
    bool bad = false;
    for (int r = 0; r < n; r++) {
        const uint8_t v = by_rank ? src[r] : src[gid_of(r)];
        bad |= (v >= D);
        pl[q.at(r)] = v;
    }
    if (bad) {
        makespan[k] = __longlong_as_double(0x7ff8000000000000LL);
        for (int j = 0; j < D; j++) {
            busy_out[(size_t)k * D + j] = 0.0;
            transfer_out[(size_t)k * D + j] = 0.0;
            peak_out[(size_t)k * D + j] = 0;
        }
        feasible[k] = 0;
        if (err) *err = 1;
        return;
    }

    for (int j = 0; j < D; j++) {
        fin_r[q.at(j)] = -1;
        busy[q.at(j)] = 0.0;
        trans[q.at(j)] = 0.0;
        peak[q.at(j)] = 0;
        qtail[q.at(j)] = 0;
    }
    for (int j = 0; j < D * D; j++) link[q.at(j)] = 0.0;

    // counts per device (segment sizes), check_memory peaks (integer, exact)
    for (int r = 0; r < n; r++) {
        const int dv = pl[q.at(r)];
        qtail[q.at(dv)] += 1;
        peak[q.at(dv)] += (long long)g.resident[r];
        left[q.at(r)] = (uint16_t)indeg_of(r);
        maxarr[q.at(r)] = 0.0;
    }
    {
        int base = 0;
        for (int j = 0; j < D; j++) {
            const int c = qtail[q.at(j)];
            qhead[q.at(j)] = (uint16_t)base;
            qtail[q.at(j)] = (uint16_t)base;
            base += c;
        }
    }
    // sources enter their device queue at t=0 in rank order (pkg/simulator.py:154-156)
    for (int r = 0; r < n; r++) {
        if (indeg_of(r) == 0) {
            const int dv = pl[q.at(r)];
            const int pos = qtail[q.at(dv)];
            devq[q.at(pos)] = (uint16_t)r;
            qtail[q.at(dv)] = (uint16_t)(pos + 1);
        }
    }

    int n_order = 0;
    int32_t *ord = order ? order + (size_t)k * n : nullptr;

    // start_next(dev, now): pkg/simulator.py:146-152
    auto start_next = [&](int dv, double now) {
        if (fin_r[q.at(dv)] >= 0) return;
        const int h = qhead[q.at(dv)];
        if (h >= qtail[q.at(dv)]) return;
        const int r = devq[q.at(h)];
        qhead[q.at(dv)] = (uint16_t)(h + 1);
        const double dur = g_dur[(size_t)r * D + dv];
        busy[q.at(dv)] += dur;
        fin_t[q.at(dv)] = now + dur;
        fin_r[q.at(dv)] = r;
        if (ord) ord[n_order++] = gid_of(r);
    };
    for (int j = 0; j < D; j++) start_next(j, 0.0);

    int n_heap = 0;
    double mk = 0.0;
    for (;;) {
        // next FINISH: min (t, rank) over busy devices
        int bd = -1, br = 0;
        double bt = 0.0;
        for (int j = 0; j < D; j++) {
            const int r = fin_r[q.at(j)];
            if (r >= 0) {
                const double t = fin_t[q.at(j)];
                if (bd < 0 || key_less(t, r, bt, br)) {
                    bd = j;
                    bt = t;
                    br = r;
                }
            }
        }
        int hr = 0;
        double ht = 0.0;
        if (n_heap > 0) {
            hr = heap[q.at(0)];
            ht = maxarr[q.at(hr)];
        }
        if (bd >= 0 && (n_heap == 0 || bt <= ht)) {
            // ---- FINISH (pkg/simulator.py:162-178) ----
            fin_r[q.at(bd)] = -1;
            mk = bt > mk ? bt : mk;
            const int e0 = g_off[br], e1 = g_off[br + 1];
            for (int e = e0; e < e1; e++) {
                const int dst = dst_of(e);
                const int ddev = pl[q.at(dst)];
                const double nbytes = g_bytes[e];
                double arrive;
                if (ddev == bd || nbytes == 0.0) {
                    arrive = bt;
                } else {
                    const int li = bd * D + ddev;
                    const double lf = link[q.at(li)];
                    const double begin = lf > bt ? lf : bt;
                    const double dur = nbytes / g_bw[li];
                    const double end = begin + dur;
                    link[q.at(li)] = end;
                    trans[q.at(bd)] += dur;
                    arrive = end;
                }
                const double ma = maxarr[q.at(dst)];
                maxarr[q.at(dst)] = arrive > ma ? arrive : ma;
                const int l = left[q.at(dst)] - 1;
                left[q.at(dst)] = (uint16_t)l;
                if (l == 0) {
                    // READY(dst) with key (maxarr, 1, rank): heap push
                    const double t = maxarr[q.at(dst)];
                    int i = n_heap++;
                    while (i > 0) {
                        const int p = (i - 1) >> 1;
                        const int pr = heap[q.at(p)];
                        if (!key_less(t, dst, maxarr[q.at(pr)], pr)) break;
                        heap[q.at(i)] = (uint16_t)pr;
                        i = p;
                    }
                    heap[q.at(i)] = (uint16_t)dst;
                }
            }
            start_next(bd, bt);
        } else if (n_heap > 0) {
            // ---- READY (= the reference's final ARRIVAL, pkg/simulator.py:179-184) ----
            const int last = heap[q.at(--n_heap)];
            if (n_heap > 0) {
                const double xt = maxarr[q.at(last)];
                int i = 0;
                for (;;) {
                    int c = 2 * i + 1;
                    if (c >= n_heap) break;
                    int cr = heap[q.at(c)];
                    double ct = maxarr[q.at(cr)];
                    if (c + 1 < n_heap) {
                        const int c2 = heap[q.at(c + 1)];
                        const double t2 = maxarr[q.at(c2)];
                        if (key_less(t2, c2, ct, cr)) {
                            c++;
                            cr = c2;
                            ct = t2;
                        }
                    }
                    if (!key_less(ct, cr, xt, last)) break;
                    heap[q.at(i)] = (uint16_t)cr;
                    i = c;
                }
                heap[q.at(i)] = (uint16_t)last;
            }
            const int dv = pl[q.at(hr)];
            // sorted insertion into the device queue (tail, usually O(1))
            int pos = qtail[q.at(dv)];
            const int h = qhead[q.at(dv)];
            while (pos > h) {
                const int pr = devq[q.at(pos - 1)];
                if (!key_less(ht, hr, maxarr[q.at(pr)], pr)) break;
                devq[q.at(pos)] = (uint16_t)pr;
                pos--;
            }
            devq[q.at(pos)] = (uint16_t)hr;
            qtail[q.at(dv)] = (uint16_t)(qtail[q.at(dv)] + 1);
            start_next(dv, ht);
        } else {
            break;
        }
    }

    makespan[k] = mk;
    bool ok = true;
    for (int j = 0; j < D; j++) {
        busy_out[(size_t)k * D + j] = busy[q.at(j)];
        transfer_out[(size_t)k * D + j] = trans[q.at(j)];
        const long long pk = peak[q.at(j)];
        peak_out[(size_t)k * D + j] = pk;
        ok &= pk <= (long long)g.mem[j];
    }
    feasible[k] = ok ? 1 : 0;
}

size_t slot_bytes(int n, int d) {
    size_t b = (size_t)n * 8 + (size_t)d * 8 * 4 + (size_t)d * d * 8 + (size_t)d * 8;  // f64/i64
    b += (size_t)d * 4;                                                                  // fin_r
    b += (size_t)n * 2 * 3 + (size_t)d * 2 * 2;                                          // u16
    b += (size_t)n;                                                                      // u8
    return b;
}

constexpr size_t kSmemBudget = 220 * 1024;

}  // namespace

extern "C" int dp_graph_create(int32_t n, int32_t d, const double *h_cost, const int32_t *h_indeg,
                               const int32_t *h_out_off, const int32_t *h_out_dst, const int64_t *h_out_bytes,
                               const int64_t *h_resident, const int32_t *h_gid, const double *h_rate,
                               const double *h_bw, const int64_t *h_mem, dp_graph **out) {
    DP_ENTRY();
    DP_REQUIRE(out != nullptr, "dp_graph_create: out is NULL");
    DP_REQUIRE(n >= 0 && n < 65536, "dp_graph_create: need 0 <= n < 65536 groups");
    DP_REQUIRE(d >= 1 && d <= 32, "dp_graph_create: need 1 <= d <= 32 devices");
    const int e = h_out_off[n];
    DP_REQUIRE(e >= 0, "dp_graph_create: bad CSR");
    int max_indeg = 0;
    for (int r = 0; r < n; r++) {
        DP_REQUIRE(h_indeg[r] >= 0 && h_indeg[r] < 65536, "dp_graph_create: in-degree out of range");
        max_indeg = h_indeg[r] > max_indeg ? h_indeg[r] : max_indeg;
    }
    std::string why;
    dp_graph *g = new dp_graph();
    g->n = n;
    g->d = d;
    g->e = e;
    g->max_indeg = max_indeg;
    g->sim_smem_per_placement = slot_bytes(n, d);
    double *h_dur = new double[(size_t)(n > 0 ? n : 1) * d];
    for (int r = 0; r < n; r++)
        for (int j = 0; j < d; j++) h_dur[(size_t)r * d + j] = h_cost[r] / h_rate[j];
    double *h_b = new double[e > 0 ? e : 1];
    for (int i = 0; i < e; i++) h_b[i] = (double)h_out_bytes[i];
    int32_t *h_rank = new int32_t[n > 0 ? n : 1];
    for (int r = 0; r < n; r++) h_rank[h_gid[r]] = r;

    auto up = [&](void **dst, const void *srcp, size_t bytes) -> bool {
        if (bytes == 0) bytes = 8;
        if (cudaMalloc(dst, bytes) != cudaSuccess) return false;
        if (srcp && cudaMemcpy(*dst, srcp, bytes, cudaMemcpyHostToDevice) != cudaSuccess) return false;
        return true;
    };
    bool ok = up((void **)&g->cost, n ? h_cost : nullptr, sizeof(double) * n) &&
              up((void **)&g->dur, h_dur, sizeof(double) * n * d) &&
              up((void **)&g->indeg, n ? h_indeg : nullptr, sizeof(int32_t) * n) &&
              up((void **)&g->out_off, h_out_off, sizeof(int32_t) * (n + 1)) &&
              up((void **)&g->out_dst, e ? h_out_dst : nullptr, sizeof(int32_t) * e) &&
              up((void **)&g->out_bytes, e ? h_b : nullptr, sizeof(double) * e) &&
              up((void **)&g->resident, n ? h_resident : nullptr, sizeof(int64_t) * n) &&
              up((void **)&g->gid, n ? h_gid : nullptr, sizeof(int32_t) * n) &&
              up((void **)&g->rank, n ? h_rank : nullptr, sizeof(int32_t) * n) &&
              up((void **)&g->rate, h_rate, sizeof(double) * d) &&
              up((void **)&g->bw, h_bw, sizeof(double) * d * d) &&
              up((void **)&g->mem, h_mem, sizeof(int64_t) * d);
    delete[] h_dur;
    delete[] h_b;
    delete[] h_rank;
    if (!ok) {
        dp::set_error(std::string("dp_graph_create: ") + cudaGetErrorString(cudaGetLastError()));
        dp_graph_destroy(g);
        return DP_ECUDA;
    }
    *out = g;
    return DP_OK;
}

extern "C" void dp_graph_destroy(dp_graph *g) {
    if (!g) return;
    void *ptrs[] = {g->cost, g->dur, g->indeg, g->out_off, g->out_dst, g->out_bytes,
                    g->resident, g->gid, g->rank, g->rate, g->bw, g->mem};
    for (void *p : ptrs)
        if (p) cudaFree(p);
    (void)cudaGetLastError();
    delete g;
}

extern "C" int dp_simulate_batch(const dp_graph *g, int32_t K, const uint8_t *placement, int32_t by_rank,
                                 double *makespan, double *busy, double *transfer, int64_t *peak,
                                 uint8_t *feasible, int32_t *order, uint8_t *err, void *stream) {
    DP_ENTRY();
    DP_REQUIRE(g != nullptr, "dp_simulate_batch: graph is NULL");
    DP_REQUIRE(K >= 0, "dp_simulate_batch: K < 0");
    if (K == 0) return DP_OK;
    const size_t per = g->sim_smem_per_placement;
    const size_t gb = graph_smem_bytes(g->n, g->d, g->e);
    // stage the graph in shared memory when it leaves room for the placements
    const bool gs = gb <= kSmemBudget / 2 && (kSmemBudget - gb) / per >= 1;
    int s_max = (int)((kSmemBudget - (gs ? gb : 0)) / per);
    if (s_max > 128) s_max = 128;
    DP_REQUIRE(s_max >= 1, "dp_simulate_batch: graph too large for the shared-memory simulator");
    // spread small batches over all SMs; pack large ones
    int S = dp::ceil_div(K, dp::kNumSMs);
    if (S > s_max) S = s_max;
    if (S < 1) S = 1;
    const int grid = dp::ceil_div(K, S);
    const size_t smem = per * S + (gs ? gb : 0) + 16;
    const void *fn = gs ? (const void *)sim_kernel<true> : (const void *)sim_kernel<false>;
    if (smem > 48 * 1024) DP_CUDA_TRY(dp::allow_big_smem(fn, smem));
    const int threads = ((S + 31) / 32) * 32;
    if (gs)
        sim_kernel<true><<<grid, threads, smem, (cudaStream_t)stream>>>(*g, K, placement, by_rank, makespan, busy,
                                                                        transfer, peak, feasible, order, err, S);
    else
        sim_kernel<false><<<grid, threads, smem, (cudaStream_t)stream>>>(*g, K, placement, by_rank, makespan, busy,
                                                                         transfer, peak, feasible, order, err, S);
    DP_LAUNCH_CHECK();
    return DP_OK;
}
