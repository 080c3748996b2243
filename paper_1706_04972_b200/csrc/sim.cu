// K-sim: batched, event-exact placement simulator (sm_100a).
//
// Replaces simulate()/check_memory() of the reference cost model,
// /root/reference/pkg/src/devplace/simulator.py:93-194, for K placements per
// launch.  One thread owns one placement; its event state lives in shared
// memory (SoA, slot-interleaved so lanes at the same step touch consecutive
// words) and, for D <= 8 devices, its per-device state (pending FINISH slot,
// ready-queue bounds, busy/transfer/peak accumulators) in registers.  The
// graph (CSR by topo rank, durations, bytes, bandwidths) is staged once per
// CTA in shared memory when it fits, else read through L1/L2.
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

#include <cstring>
#include <vector>

#include "common.cuh"
#include "tc.cuh"

namespace {

__device__ __forceinline__ bool key_less(double ta, int ra, double tb, int rb) {
    return ta < tb || (ta == tb && ra < rb);
}

// Per-device state, register-resident (DM >= D): runtime indices resolve to
// unrolled predicated selects instead of shared-memory round trips.
template <int DM>
struct DevRegs {
    double fin_t[DM], busy[DM], trans[DM];
    long long peak[DM];
    int fin_r[DM], qh[DM], qt[DM];
    __device__ __forceinline__ void init() {
#pragma unroll
        for (int j = 0; j < DM; j++) {
            fin_t[j] = busy[j] = trans[j] = 0.0;
            peak[j] = 0;
            fin_r[j] = -1;
            qh[j] = qt[j] = 0;
        }
    }
#define DP_GET(name, T)                                            \
    __device__ __forceinline__ T get_##name(int d) const {         \
        T v = name[0];                                             \
        _Pragma("unroll") for (int j = 1; j < DM; j++) if (j == d) v = name[j]; \
        return v;                                                  \
    }                                                              \
    __device__ __forceinline__ void set_##name(int d, T v) {       \
        _Pragma("unroll") for (int j = 0; j < DM; j++) if (j == d) name[j] = v; \
    }
    DP_GET(fin_t, double)
    DP_GET(busy, double)
    DP_GET(trans, double)
    DP_GET(peak, long long)
    DP_GET(fin_r, int)
    DP_GET(qh, int)
    DP_GET(qt, int)
#undef DP_GET
};

// Same interface, shared-memory resident (any D <= 32).
struct DevSmem {
    double *fin_t, *busy, *trans;
    long long *peak;
    int *fin_r, *qh, *qt;
    int S, s, D;
    __device__ __forceinline__ int at(int j) const { return j * S + s; }
    __device__ __forceinline__ void init() {
        for (int j = 0; j < D; j++) {
            fin_t[at(j)] = busy[at(j)] = trans[at(j)] = 0.0;
            peak[at(j)] = 0;
            fin_r[at(j)] = -1;
            qh[at(j)] = qt[at(j)] = 0;
        }
    }
#define DP_GET(name, T)                                                                  \
    __device__ __forceinline__ T get_##name(int d) const { return name[at(d)]; }         \
    __device__ __forceinline__ void set_##name(int d, T v) { name[at(d)] = v; }
    DP_GET(fin_t, double)
    DP_GET(busy, double)
    DP_GET(trans, double)
    DP_GET(peak, long long)
    DP_GET(fin_r, int)
    DP_GET(qh, int)
    DP_GET(qt, int)
#undef DP_GET
};

template <int DM>
struct DevPick {  // register state when DM > 0
    template <class A, class B>
    __device__ __forceinline__ static A &get(A &a, B &) { return a; }
};
template <>
struct DevPick<0> {  // shared-memory state
    template <class A, class B>
    __device__ __forceinline__ static B &get(A &, B &b) { return b; }
};

// Bytes of the graph image staged in shared memory (GS=true).
__host__ __device__ inline size_t graph_smem_bytes(int n, int d, int e) {
    size_t b = 8 * ((size_t)n * d + e + (size_t)d * d) + 4 * (size_t)(n + 1) + 2 * ((size_t)e + 2 * n);
    return (b + 15) & ~(size_t)15;
}

// Stage the graph image into shared memory with the TMA bulk-copy engine (one
// elected thread issues <= 32 KB chunks against one mbarrier; every thread
// waits on its phase).  The image layout is the GS carve-up below.
__device__ __forceinline__ void stage_graph(unsigned char *smem, const dp_graph &g, uint64_t *bar) {
    if (threadIdx.x == 0) {
        dp::tc::mbar_init(bar, 1);
        dp::tc::fence_mbar_init();
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        const uint32_t total = (uint32_t)g.image_bytes;
        dp::tc::mbar_expect_tx(bar, total);
        for (uint32_t o = 0; o < total; o += 32768u)
            dp::tc::bulk_load(smem + o, g.image + o, total - o < 32768u ? total - o : 32768u, bar);
    }
    dp::tc::mbar_wait(bar, 0);
}

// Per-placement shared-memory bytes (DM > 0: device state in registers).
__host__ __device__ inline size_t slot_bytes(int n, int d, bool reg_dev) {
    size_t b = (size_t)n * 8 + (size_t)d * d * 8;  // maxarr, link_free
    if (!reg_dev) b += (size_t)d * (8 * 4 + 4 + 2 * 4);  // fin_t busy trans peak | fin_r | qh qt (int)
    b += (size_t)n * 2 * 3;                        // left, heap, devq (u16)
    b += (size_t)n;                                // placement (u8)
    return (b + 7) & ~(size_t)7;
}

template <bool GS, int DM>
__global__ void __launch_bounds__(128) sim_kernel(dp_graph g, int K, const uint8_t *__restrict__ placement,
                                                  int by_rank, double *__restrict__ makespan,
                                                  double *__restrict__ busy_out, double *__restrict__ transfer_out,
                                                  int64_t *__restrict__ peak_out, uint8_t *__restrict__ feasible,
                                                  int32_t *__restrict__ order, uint8_t *__restrict__ err, int S) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ uint64_t s_stage_bar;
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
        stage_graph(smem, g, &s_stage_bar);
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
    auto at = [&](int i) -> int { return i * S + s; };

    // ---- shared-memory carve-up (all arrays slot-interleaved: [i*S + s]) ----
    double *maxarr = reinterpret_cast<double *>(smem + gbytes);  // [n]  READY time (max arrival)
    double *link = maxarr + n * S;                                // [D*D] link_free
    unsigned char *tail = reinterpret_cast<unsigned char *>(link + D * D * S);
    DevSmem ds;
    if (DM == 0) {
        ds.fin_t = reinterpret_cast<double *>(tail);
        ds.busy = ds.fin_t + D * S;
        ds.trans = ds.busy + D * S;
        ds.peak = reinterpret_cast<long long *>(ds.trans + D * S);
        ds.fin_r = reinterpret_cast<int *>(ds.peak + D * S);
        ds.qh = ds.fin_r + D * S;
        ds.qt = ds.qh + D * S;
        ds.S = S;
        ds.s = s;
        ds.D = D;
        tail = reinterpret_cast<unsigned char *>(ds.qt + D * S);
    }
    uint16_t *left = reinterpret_cast<uint16_t *>(tail);  // [n] unfinished preds
    uint16_t *heap = left + n * S;                         // [n] READY heap (ranks)
    uint16_t *devq = heap + n * S;                         // [n] ready queues
    uint8_t *pl = reinterpret_cast<uint8_t *>(devq + n * S);  // [n] device of rank
    DevRegs<(DM > 0 ? DM : 1)> dr;

    // ---- placement load + validation (pkg/simulator.py:109-116) ----
    const uint8_t *src = placement + (size_t)k * n;
    bool bad = false;
    for (int r = 0; r < n; r++) {
        const uint8_t v = by_rank ? src[r] : src[gid_of(r)];
        bad |= (v >= D);
        pl[at(r)] = v;
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
    auto &dv_ = DevPick<DM>::get(dr, ds);
    dv_.init();
    for (int j = 0; j < D * D; j++) link[at(j)] = 0.0;

    // counts per device (segment sizes), check_memory peaks (integer, exact)
    for (int r = 0; r < n; r++) {
        const int d = pl[at(r)];
        dv_.set_qt(d, dv_.get_qt(d) + 1);
        dv_.set_peak(d, dv_.get_peak(d) + (long long)g.resident[r]);
        left[at(r)] = (uint16_t)indeg_of(r);
        maxarr[at(r)] = 0.0;
    }
    {
        int base = 0;
        for (int j = 0; j < D; j++) {
            const int c = dv_.get_qt(j);
            dv_.set_qh(j, base);
            dv_.set_qt(j, base);
            base += c;
        }
    }
    // sources enter their device queue at t=0 in rank order (pkg/simulator.py:154-156)
    for (int r = 0; r < n; r++) {
        if (indeg_of(r) == 0) {
            const int d = pl[at(r)];
            const int pos = dv_.get_qt(d);
            devq[at(pos)] = (uint16_t)r;
            dv_.set_qt(d, pos + 1);
        }
    }

    int n_order = 0;
    int32_t *ord = order ? order + (size_t)k * n : nullptr;

    // start_next(dev, now): pkg/simulator.py:146-152
    auto start_next = [&](int d, double now) {
        if (dv_.get_fin_r(d) >= 0) return;
        const int h = dv_.get_qh(d);
        if (h >= dv_.get_qt(d)) return;
        const int r = devq[at(h)];
        dv_.set_qh(d, h + 1);
        const double dur = g_dur[r * D + d];
        dv_.set_busy(d, dv_.get_busy(d) + dur);
        dv_.set_fin_t(d, now + dur);
        dv_.set_fin_r(d, r);
        if (ord) ord[n_order++] = gid_of(r);
    };
    for (int j = 0; j < D; j++) start_next(j, 0.0);

    int n_heap = 0;
    double mk = 0.0;
    for (;;) {
        // next FINISH: min (t, rank) over busy devices
        int bd = -1, br = 0;
        double bt = 0.0;
        if constexpr (DM > 0) {
#pragma unroll
            for (int j = 0; j < DM; j++) {
                const int r = dr.fin_r[j];
                if (j < D && r >= 0) {
                    const double t = dr.fin_t[j];
                    if (bd < 0 || key_less(t, r, bt, br)) {
                        bd = j;
                        bt = t;
                        br = r;
                    }
                }
            }
        } else {
            for (int j = 0; j < D; j++) {
                const int r = ds.get_fin_r(j);
                if (r >= 0) {
                    const double t = ds.get_fin_t(j);
                    if (bd < 0 || key_less(t, r, bt, br)) {
                        bd = j;
                        bt = t;
                        br = r;
                    }
                }
            }
        }
        int hr = 0;
        double ht = 0.0;
        if (n_heap > 0) {
            hr = heap[at(0)];
            ht = maxarr[at(hr)];
        }
        if (bd >= 0 && (n_heap == 0 || bt <= ht)) {
            // ---- FINISH (pkg/simulator.py:162-178) ----
            dv_.set_fin_r(bd, -1);
            mk = bt > mk ? bt : mk;
            const int e0 = g_off[br], e1 = g_off[br + 1];
            double tr = 0.0;
            bool any_link = false;
            for (int e = e0; e < e1; e++) {
                const int dst = dst_of(e);
                const int ddev = pl[at(dst)];
                const double nbytes = g_bytes[e];
                double arrive;
                if (ddev == bd || nbytes == 0.0) {
                    arrive = bt;
                } else {
                    const int li = bd * D + ddev;
                    const double lf = link[at(li)];
                    const double begin = lf > bt ? lf : bt;
                    const double dur = nbytes / g_bw[li];
                    const double end = begin + dur;
                    link[at(li)] = end;
                    // transfer[dev] += dur, in edge order (sequential, same rounding)
                    tr = any_link ? tr + dur : dv_.get_trans(bd) + dur;
                    any_link = true;
                    arrive = end;
                }
                const double ma = maxarr[at(dst)];
                maxarr[at(dst)] = arrive > ma ? arrive : ma;
                const int l = left[at(dst)] - 1;
                left[at(dst)] = (uint16_t)l;
                if (l == 0) {
                    // READY(dst) with key (maxarr, 1, rank): heap push
                    const double t = maxarr[at(dst)];
                    int i = n_heap++;
                    while (i > 0) {
                        const int p = (i - 1) >> 1;
                        const int pr = heap[at(p)];
                        if (!key_less(t, dst, maxarr[at(pr)], pr)) break;
                        heap[at(i)] = (uint16_t)pr;
                        i = p;
                    }
                    heap[at(i)] = (uint16_t)dst;
                }
            }
            if (any_link) dv_.set_trans(bd, tr);
            start_next(bd, bt);
        } else if (n_heap > 0) {
            // ---- READY (= the reference's final ARRIVAL, pkg/simulator.py:179-184) ----
            const int last = heap[at(--n_heap)];
            if (n_heap > 0) {
                const double xt = maxarr[at(last)];
                int i = 0;
                for (;;) {
                    int c = 2 * i + 1;
                    if (c >= n_heap) break;
                    int cr = heap[at(c)];
                    double ct = maxarr[at(cr)];
                    if (c + 1 < n_heap) {
                        const int c2 = heap[at(c + 1)];
                        const double t2 = maxarr[at(c2)];
                        if (key_less(t2, c2, ct, cr)) {
                            c++;
                            cr = c2;
                            ct = t2;
                        }
                    }
                    if (!key_less(ct, cr, xt, last)) break;
                    heap[at(i)] = (uint16_t)cr;
                    i = c;
                }
                heap[at(i)] = (uint16_t)last;
            }
            const int d = pl[at(hr)];
            // sorted insertion into the device queue (tail, usually O(1))
            const int qt = dv_.get_qt(d);
            int pos = qt;
            const int h = dv_.get_qh(d);
            while (pos > h) {
                const int pr = devq[at(pos - 1)];
                if (!key_less(ht, hr, maxarr[at(pr)], pr)) break;
                devq[at(pos)] = (uint16_t)pr;
                pos--;
            }
            devq[at(pos)] = (uint16_t)hr;
            dv_.set_qt(d, qt + 1);
            start_next(d, ht);
        } else {
            break;
        }
    }

    makespan[k] = mk;
    bool ok = true;
    for (int j = 0; j < D; j++) {
        busy_out[(size_t)k * D + j] = dv_.get_busy(j);
        transfer_out[(size_t)k * D + j] = dv_.get_trans(j);
        const long long pk = dv_.get_peak(j);
        peak_out[(size_t)k * D + j] = pk;
        ok &= pk <= (long long)g.mem[j];
    }
    feasible[k] = ok ? 1 : 0;
}

// ---------------------------------------------------------------- warp per placement
// One warp scores one placement (the north-star K-sim design) — the latency
// path for small K; the CTA's warps share the graph image staged in shared
// memory.  Lane d (< D) keeps device d's state in registers (pending FINISH,
// ready-queue bounds, busy / transfer / peak).  The next event is a warp
// shuffle argmin over the devices' FINISH keys against the READY-heap top.  A
// FINISH's out-edges go lane-parallel (link durations — the fp64 divisions —
// arrival max-reduction into maxarr, in-degree countdown); only the link-queue
// chain (link_free, transfer[dev] += dur) is walked in edge order, and heap
// updates are executed redundantly by every lane (broadcast reads) with lane 0
// writing.  Same event semantics and fp64 operation order as sim_kernel
// (SURVEY.md Appendix A.2): bit-identical outputs, dispatch order included.
constexpr int kSimWarps = 16;  // max warps per CTA (placements sharing one staged graph)

__host__ __device__ inline size_t warp_slot_bytes(int n, int d) {
    size_t b = (size_t)n * 8 + (size_t)d * d * 8;  // maxarr, link_free
    b += (size_t)n * 2 * 3;                        // left, heap, devq (u16)
    b += (size_t)n;                                // placement (u8)
    return (b + 15) & ~(size_t)15;
}

template <bool GS>
__global__ void __launch_bounds__(32 * kSimWarps) sim_warp_kernel(
    dp_graph g, int K, const uint8_t *__restrict__ placement, int by_rank, double *__restrict__ makespan,
    double *__restrict__ busy_out, double *__restrict__ transfer_out, int64_t *__restrict__ peak_out,
    uint8_t *__restrict__ feasible, int32_t *__restrict__ order, uint8_t *__restrict__ err) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ uint64_t s_stage_bar;
    constexpr unsigned kFull = 0xffffffffu;
    const int tid = threadIdx.x, lane = tid & 31, wp = tid >> 5;
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
        stage_graph(smem, g, &s_stage_bar);
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
    const int k = blockIdx.x * (blockDim.x >> 5) + wp;
    if (k >= K) return;  // whole warps only; no CTA barrier follows
    unsigned char *base = smem + gbytes + (size_t)wp * warp_slot_bytes(n, D);
    double *maxarr = reinterpret_cast<double *>(base);  // [n] READY time (max arrival)
    double *link = maxarr + n;                          // [D*D] link_free
    uint16_t *left = reinterpret_cast<uint16_t *>(link + D * D);
    uint16_t *heap = left + n;
    uint16_t *devq = heap + n;
    uint8_t *pl = reinterpret_cast<uint8_t *>(devq + n);
    const unsigned lt_mask = (1u << lane) - 1u;

    // ---- placement load + validation (pkg/simulator.py:109-116) ----
    const uint8_t *src = placement + (size_t)k * n;
    bool bad = false;
    for (int r = lane; r < n; r += 32) {
        const uint8_t v = by_rank ? src[r] : src[gid_of(r)];
        bad |= (v >= D);
        pl[r] = v;
        left[r] = (uint16_t)indeg_of(r);
        maxarr[r] = 0.0;
    }
    if (__any_sync(kFull, bad)) {
        if (lane == 0) {
            makespan[k] = __longlong_as_double(0x7ff8000000000000LL);
            feasible[k] = 0;
            if (err) *err = 1;
        }
        for (int j = lane; j < D; j += 32) {
            busy_out[(size_t)k * D + j] = 0.0;
            transfer_out[(size_t)k * D + j] = 0.0;
            peak_out[(size_t)k * D + j] = 0;
        }
        return;
    }
    for (int j = lane; j < D * D; j += 32) link[j] = 0.0;
    __syncwarp();
    // ---- per-device counts and check_memory peaks (integer, exact) -> lane d ----
    int qh = 0, qt = 0;
    long long pk = 0;
    for (int d = 0; d < D; d++) {
        int c = 0;
        long long p = 0;
        for (int r = lane; r < n; r += 32)
            if (pl[r] == d) {
                c++;
                p += (long long)g.resident[r];
            }
        c = __reduce_add_sync(kFull, c);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) p += __shfl_xor_sync(kFull, p, o);
        if (lane == d) {
            qt = c;
            pk = p;
        }
    }
    {
        // exclusive prefix over devices -> queue segment bases
        int incl = lane < D ? qt : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int v = __shfl_up_sync(kFull, incl, o);
            if (lane >= o) incl += v;
        }
        qh = qt = incl - (lane < D ? qt : 0);
    }
    // sources enter their device queue at t=0 in rank order (pkg/simulator.py:154-156)
    for (int c0 = 0; c0 < n; c0 += 32) {
        const int r = c0 + lane;
        const int dv = (r < n && left[r] == 0) ? (int)pl[r] : -1;
        for (int d = 0; d < D; d++) {
            const unsigned m = __ballot_sync(kFull, dv == d);
            if (!m) continue;
            const int qd = __shfl_sync(kFull, qt, d);
            if (dv == d) devq[qd + __popc(m & lt_mask)] = (uint16_t)r;
            if (lane == d) qt += __popc(m);
        }
    }
    __syncwarp();
    double fin_t = 0.0, busy = 0.0, trans = 0.0;
    int fin_r = -1;
    int n_order = 0;
    int32_t *ord = order ? order + (size_t)k * n : nullptr;
    // start_next(dev, now) on the lanes that ask, device order for the dispatch log (pkg/simulator.py:146-152)
    auto start_next = [&](bool want, double now) {
        const bool go = want && lane < D && fin_r < 0 && qh < qt;
        const unsigned m = __ballot_sync(kFull, go);
        if (go) {
            const int r = devq[qh];
            qh++;
            const double du = g_dur[r * D + lane];
            busy += du;
            fin_t = now + du;
            fin_r = r;
            if (ord) ord[n_order + __popc(m & lt_mask)] = gid_of(r);
        }
        n_order += __popc(m);
    };
    start_next(true, 0.0);
    int d_pow2 = 1;
    while (d_pow2 < D) d_pow2 <<= 1;
    int n_heap = 0;
    double mk = 0.0;
    for (;;) {
        // next FINISH: min (t, rank) over busy devices (shuffle argmin)
        const bool act = lane < D && fin_r >= 0;
        double bt = act ? fin_t : 0.0;
        int br = act ? fin_r : -1, bd = lane;
        for (int o = d_pow2 >> 1; o > 0; o >>= 1) {
            const double ot = __shfl_xor_sync(kFull, bt, o);
            const int orr = __shfl_xor_sync(kFull, br, o), od = __shfl_xor_sync(kFull, bd, o);
            if (orr >= 0 && (br < 0 || key_less(ot, orr, bt, br))) {
                bt = ot;
                br = orr;
                bd = od;
            }
        }
        bt = __shfl_sync(kFull, bt, 0);
        br = __shfl_sync(kFull, br, 0);
        bd = __shfl_sync(kFull, bd, 0);
        int hr = 0;
        double ht = 0.0;
        if (n_heap > 0) {
            hr = heap[0];
            ht = maxarr[hr];
        }
        if (br >= 0 && (n_heap == 0 || bt <= ht)) {
            // ---- FINISH (pkg/simulator.py:162-178) ----
            if (lane == bd) fin_r = -1;
            mk = bt > mk ? bt : mk;
            const int e0 = g_off[br], e1 = g_off[br + 1];
            double tr = __shfl_sync(kFull, trans, bd);
            for (int eb = e0; eb < e1; eb += 32) {
                const int e = eb + lane;
                const bool has = e < e1;
                int dst = 0, ddev = 0;
                double dur = 0.0;
                bool lk = false;
                if (has) {
                    dst = dst_of(e);
                    ddev = pl[dst];
                    const double nbytes = g_bytes[e];
                    lk = ddev != bd && nbytes != 0.0;
                    if (lk) dur = nbytes / g_bw[bd * D + ddev];
                }
                double arrive = bt;
                // link queues in edge order: begin = max(t, link_free), transfer[dev] += dur
                unsigned lm = __ballot_sync(kFull, lk);
                while (lm) {
                    const int j = __ffs(lm) - 1;
                    lm &= lm - 1;
                    const int li = bd * D + __shfl_sync(kFull, ddev, j);
                    const double dj = __shfl_sync(kFull, dur, j);
                    const double lf = link[li];
                    const double begin = lf > bt ? lf : bt;
                    const double end = begin + dj;
                    __syncwarp();
                    if (lane == 0) link[li] = end;
                    __syncwarp();
                    tr = tr + dj;
                    if (lane == j) arrive = end;
                }
                // arrivals fold into maxarr, in-degrees count down (one edge per dst: lane-parallel)
                bool ready = false;
                if (has) {
                    const double ma = maxarr[dst];
                    maxarr[dst] = arrive > ma ? arrive : ma;
                    const int l = left[dst] - 1;
                    left[dst] = (uint16_t)l;
                    ready = l == 0;
                }
                __syncwarp();
                // READY pushes, key (maxarr, rank): keys are unique, so push order is immaterial
                unsigned rm = __ballot_sync(kFull, ready);
                while (rm) {
                    const int j = __ffs(rm) - 1;
                    rm &= rm - 1;
                    const int r = __shfl_sync(kFull, dst, j);
                    const double t = maxarr[r];
                    int i = n_heap++;
                    while (i > 0) {
                        const int p = (i - 1) >> 1;
                        const int pr = heap[p];
                        if (!key_less(t, r, maxarr[pr], pr)) break;
                        __syncwarp();  // every lane has read heap[p] before lane 0 moves entries
                        if (lane == 0) heap[i] = (uint16_t)pr;
                        i = p;
                    }
                    if (lane == 0) heap[i] = (uint16_t)r;
                    __syncwarp();
                }
            }
            if (lane == bd) trans = tr;
            start_next(lane == bd, bt);
        } else if (n_heap > 0) {
            // ---- READY (= the reference's final ARRIVAL, pkg/simulator.py:179-184) ----
            const int last = heap[--n_heap];
            __syncwarp();  // every lane's reads of heap[0] / heap[last] precede lane 0's writes below
            if (n_heap > 0) {
                const double xt = maxarr[last];
                int i = 0;
                for (;;) {
                    int c = 2 * i + 1;
                    if (c >= n_heap) break;
                    int cr = heap[c];
                    double ct = maxarr[cr];
                    if (c + 1 < n_heap) {
                        const int c2 = heap[c + 1];
                        const double t2 = maxarr[c2];
                        if (key_less(t2, c2, ct, cr)) {
                            c++;
                            cr = c2;
                            ct = t2;
                        }
                    }
                    if (!key_less(ct, cr, xt, last)) break;
                    __syncwarp();  // reads of heap[c], heap[c+1] precede lane 0's write
                    if (lane == 0) heap[i] = (uint16_t)cr;
                    i = c;
                }
                if (lane == 0) heap[i] = (uint16_t)last;
            }
            __syncwarp();
            const int d = pl[hr];
            // sorted insertion into the device queue (tail, usually O(1))
            const int qtd = __shfl_sync(kFull, qt, d), qhd = __shfl_sync(kFull, qh, d);
            int pos = qtd;
            while (pos > qhd) {
                const int pr = devq[pos - 1];
                if (!key_less(ht, hr, maxarr[pr], pr)) break;
                __syncwarp();  // every lane has read devq[pos - 1] before lane 0 shifts it
                if (lane == 0) devq[pos] = (uint16_t)pr;
                pos--;
            }
            if (lane == 0) devq[pos] = (uint16_t)hr;
            __syncwarp();
            if (lane == d) qt++;
            start_next(lane == d, ht);
        } else {
            break;
        }
    }
    if (lane == 0) makespan[k] = mk;
    bool ok = true;
    if (lane < D) {
        busy_out[(size_t)k * D + lane] = busy;
        transfer_out[(size_t)k * D + lane] = trans;
        peak_out[(size_t)k * D + lane] = pk;
        ok = pk <= (long long)g.mem[lane];
    }
    ok = __all_sync(kFull, ok);
    if (lane == 0) feasible[k] = ok ? 1 : 0;
}

// Lexicographic enumeration for brute force (itertools.product order:
// the last group varies fastest), placements by gid.
__global__ void enumerate_kernel(int n, int d, unsigned long long start, int count, uint8_t *__restrict__ out) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= count) return;
    unsigned long long c = start + (unsigned long long)k;
    uint8_t *o = out + (size_t)k * n;
    for (int g = n - 1; g >= 0; g--) {
        o[g] = (uint8_t)(c % (unsigned long long)d);
        c /= (unsigned long long)d;
    }
}

// First (lowest index) minimal makespan among feasible placements, folded
// into (best_val, best_idx) with a strict < so earlier batches win ties —
// the reference's sequential `if makespan < best` (pkg/baselines.py:246-272).
__global__ void argmin_feasible_kernel(int K, const double *__restrict__ makespan, const uint8_t *__restrict__ feasible,
                                       long long base_index, double *best_val, long long *best_idx) {
    __shared__ double sv[1024];
    __shared__ long long si[1024];
    const int tid = threadIdx.x;
    double v = INFINITY;
    long long idx = -1;
    for (int k = tid; k < K; k += blockDim.x) {
        if (!feasible[k]) continue;
        const double m = makespan[k];
        if (idx < 0 || m < v) {  // k ascending per thread: first minimum kept
            v = m;
            idx = base_index + k;
        }
    }
    sv[tid] = v;
    si[tid] = idx;
    __syncthreads();
    for (int s = blockDim.x / 2; s > 0; s >>= 1) {
        if (tid < s) {
            const double v2 = sv[tid + s];
            const long long i2 = si[tid + s];
            if (i2 >= 0 && (si[tid] < 0 || v2 < sv[tid] || (v2 == sv[tid] && i2 < si[tid]))) {
                sv[tid] = v2;
                si[tid] = i2;
            }
        }
        __syncthreads();
    }
    if (tid == 0 && si[0] >= 0 && (*best_idx < 0 || sv[0] < *best_val)) {
        *best_val = sv[0];
        *best_idx = si[0];
    }
}

constexpr size_t kSmemBudget = 220 * 1024;
constexpr int kRegDevMax = 8;

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
    dp_graph *g = new dp_graph();
    g->n = n;
    g->d = d;
    g->e = e;
    g->max_indeg = max_indeg;
    g->sim_smem_per_placement = slot_bytes(n, d, d <= kRegDevMax);
    double *h_dur = new double[(size_t)(n > 0 ? n : 1) * d];
    for (int r = 0; r < n; r++)
        for (int j = 0; j < d; j++) h_dur[(size_t)r * d + j] = h_cost[r] / h_rate[j];
    double *h_b = new double[e > 0 ? e : 1];
    for (int i = 0; i < e; i++) h_b[i] = (double)h_out_bytes[i];
    int32_t *h_rank = new int32_t[n > 0 ? n : 1];
    for (int r = 0; r < n; r++) h_rank[h_gid[r]] = r;
    // shared-memory image for the TMA bulk staging (graph_smem_bytes layout)
    g->image_bytes = graph_smem_bytes(n, d, e);
    std::vector<unsigned char> img(g->image_bytes, 0);
    {
        double *idur = reinterpret_cast<double *>(img.data());
        double *ibytes = idur + (size_t)n * d;
        double *ibw = ibytes + e;
        int32_t *ioff = reinterpret_cast<int32_t *>(ibw + (size_t)d * d);
        uint16_t *idst = reinterpret_cast<uint16_t *>(ioff + n + 1);
        uint16_t *igid = idst + e;
        uint16_t *iind = igid + n;
        std::memcpy(idur, h_dur, sizeof(double) * n * d);
        std::memcpy(ibytes, h_b, sizeof(double) * e);
        std::memcpy(ibw, h_bw, sizeof(double) * d * d);
        std::memcpy(ioff, h_out_off, sizeof(int32_t) * (n + 1));
        for (int i = 0; i < e; i++) idst[i] = (uint16_t)h_out_dst[i];
        for (int r = 0; r < n; r++) {
            igid[r] = (uint16_t)h_gid[r];
            iind[r] = (uint16_t)h_indeg[r];
        }
    }

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
              up((void **)&g->mem, h_mem, sizeof(int64_t) * d) &&
              up((void **)&g->image, img.data(), g->image_bytes);
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
                    g->resident, g->gid, g->rank, g->rate, g->bw, g->mem, g->image};
    for (void *p : ptrs)
        if (p) cudaFree(p);
    (void)cudaGetLastError();
    delete g;
}

template <bool GS, int DM>
static int launch_sim(const dp_graph *g, int grid, int threads, size_t smem, cudaStream_t st, int K,
                      const uint8_t *placement, int by_rank, double *makespan, double *busy, double *transfer,
                      int64_t *peak, uint8_t *feasible, int32_t *order, uint8_t *err, int S) {
    if (smem > 48 * 1024) DP_CUDA_TRY(dp::allow_big_smem((const void *)sim_kernel<GS, DM>, smem));
    sim_kernel<GS, DM><<<grid, threads, smem, st>>>(*g, K, placement, by_rank, makespan, busy, transfer, peak,
                                                    feasible, order, err, S);
    DP_LAUNCH_CHECK();
    return DP_OK;
}

static int g_sim_variant = 0;  // dp_debug_sim_variant
extern "C" int dp_debug_sim_variant(int32_t mode) {
    DP_ENTRY();
    DP_REQUIRE(mode >= 0 && mode <= 2, "dp_debug_sim_variant: mode must be 0, 1 or 2");
    g_sim_variant = mode;
    return DP_OK;
}

// Kernel choice (measured, profiles/r01_sim_throughput.txt): one warp per
// placement everywhere except many placements of small graphs, where one
// thread per placement keeps 32x more placements in flight per warp (C1 at
// K=65536: 42M/s vs 29M/s).
inline bool sim_warp_preferred(const dp_graph *g, int K) { return !(g->n <= 128 && K >= 32768); }

template <bool GS>
static int launch_sim_warp(const dp_graph *g, int K, size_t gb, cudaStream_t st, const uint8_t *placement,
                           int by_rank, double *makespan, double *busy, double *transfer, int64_t *peak,
                           uint8_t *feasible, int32_t *order, uint8_t *err) {
    // With the graph staged, up to 16 warps share one copy and the batch is
    // packed onto <= ~20 SMs: in the training step the scorer runs beside the
    // attention backward, whose 1-CTA-per-SM tiles leave 20 SMs free
    // (att_grid) — a scorer CTA on any other SM would block one of them.
    // Without staging (large graphs): 1-warp CTAs, more resident per SM.
    int W = 1;
    if (GS) {
        W = dp::ceil_div(K, 20);
        W = W < 4 ? 4 : W > kSimWarps ? kSimWarps : W;
        const size_t per = warp_slot_bytes(g->n, g->d);
        while (W > 1 && per * W + gb + 16 > kSmemBudget) W--;
    }
    const size_t smem = warp_slot_bytes(g->n, g->d) * W + (GS ? gb : 0) + 16;
    if (smem > 48 * 1024) DP_CUDA_TRY(dp::allow_big_smem((const void *)sim_warp_kernel<GS>, smem));
    sim_warp_kernel<GS><<<dp::ceil_div(K, W), 32 * W, smem, st>>>(
        *g, K, placement, by_rank, makespan, busy, transfer, peak, feasible, order, err);
    DP_LAUNCH_CHECK();
    return DP_OK;
}

extern "C" int dp_simulate_batch(const dp_graph *g, int32_t K, const uint8_t *placement, int32_t by_rank,
                                 double *makespan, double *busy, double *transfer, int64_t *peak,
                                 uint8_t *feasible, int32_t *order, uint8_t *err, void *stream) {
    DP_ENTRY();
    DP_REQUIRE(g != nullptr, "dp_simulate_batch: graph is NULL");
    DP_REQUIRE(K >= 0, "dp_simulate_batch: K < 0");
    if (K == 0) return DP_OK;
    {
        const size_t gb = graph_smem_bytes(g->n, g->d, g->e);
        const size_t ws = warp_slot_bytes(g->n, g->d) * 4;
        const bool fits_gs = gb + ws + 16 <= kSmemBudget;
        const bool fits = warp_slot_bytes(g->n, g->d) + 16 <= kSmemBudget;
        const bool want = g_sim_variant == 1 || (g_sim_variant == 0 && sim_warp_preferred(g, K));
        if (want && fits) {
            cudaStream_t st = (cudaStream_t)stream;
            if (fits_gs)
                return launch_sim_warp<true>(g, K, gb, st, placement, by_rank, makespan, busy, transfer, peak,
                                             feasible, order, err);
            return launch_sim_warp<false>(g, K, gb, st, placement, by_rank, makespan, busy, transfer, peak,
                                          feasible, order, err);
        }
    }
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
    const int threads = ((S + 31) / 32) * 32;
    cudaStream_t st = (cudaStream_t)stream;
    const bool reg = g->d <= kRegDevMax;
    if (gs && reg)
        return launch_sim<true, kRegDevMax>(g, grid, threads, smem, st, K, placement, by_rank, makespan, busy,
                                            transfer, peak, feasible, order, err, S);
    if (gs)
        return launch_sim<true, 0>(g, grid, threads, smem, st, K, placement, by_rank, makespan, busy, transfer,
                                   peak, feasible, order, err, S);
    if (reg)
        return launch_sim<false, kRegDevMax>(g, grid, threads, smem, st, K, placement, by_rank, makespan, busy,
                                             transfer, peak, feasible, order, err, S);
    return launch_sim<false, 0>(g, grid, threads, smem, st, K, placement, by_rank, makespan, busy, transfer, peak,
                                feasible, order, err, S);
}

extern "C" int dp_enumerate_placements(int32_t n, int32_t d, uint64_t start, int32_t count, uint8_t *out,
                                       void *stream) {
    DP_ENTRY();
    DP_REQUIRE(n >= 1 && d >= 1 && d <= 255 && count >= 0 && out, "dp_enumerate_placements: bad argument");
    if (count == 0) return DP_OK;
    enumerate_kernel<<<dp::ceil_div(count, 256), 256, 0, (cudaStream_t)stream>>>(n, d, start, count, out);
    DP_LAUNCH_CHECK();
    return DP_OK;
}

extern "C" int dp_argmin_feasible(int32_t K, const double *makespan, const uint8_t *feasible, int64_t base_index,
                                  double *best_val, int64_t *best_idx, void *stream) {
    DP_ENTRY();
    DP_REQUIRE(K >= 0 && makespan && feasible && best_val && best_idx, "dp_argmin_feasible: NULL argument");
    if (K == 0) return DP_OK;
    argmin_feasible_kernel<<<1, 1024, 0, (cudaStream_t)stream>>>(K, makespan, feasible, base_index, best_val,
                                                                  (long long *)best_idx);
    DP_LAUNCH_CHECK();
    return DP_OK;
}
