/*
 * TEST INFRASTRUCTURE ONLY — CPU restatement of the reference execution-time
 * simulator, used as the parity checker for the CUDA kernel (csrc/sim.cu) and
 * as the timed CPU baseline in bench.py.  Never linked into the product.
 *
 * Follows /root/reference/pkg/src/devplace/simulator.py exactly:
 *   check_memory            simulator.py:93-106
 *   simulate                simulator.py:122-194
 *     start_next            simulator.py:146-152
 *     source seeding        simulator.py:154-158
 *     event loop            simulator.py:160-184 (heap key (t, kind, rank, gid),
 *                           FINISH=0 < ARRIVAL=1, simulator.py:119, 137)
 *     out-edges by dst rank simulator.py:139-144
 * Event heap and per-device ready heaps are binary min-heaps over the same
 * tuple keys as Python's heapq, so the pop sequence (and hence every fp64
 * operation's order) is identical.
 *
 * Graph arrays are indexed by group id (gid); out-edges are CSR by source gid
 * with each row already sorted by destination topo rank.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct { double t; int kind, rank, gid; } ev_t;
typedef struct { double t; int rank, gid; } rq_t;

static int ev_less(const ev_t *a, const ev_t *b) {
    if (a->t != b->t) return a->t < b->t;
    if (a->kind != b->kind) return a->kind < b->kind;
    if (a->rank != b->rank) return a->rank < b->rank;
    return a->gid < b->gid;
}
static int rq_less(const rq_t *a, const rq_t *b) {
    if (a->t != b->t) return a->t < b->t;
    if (a->rank != b->rank) return a->rank < b->rank;
    return a->gid < b->gid;
}

#define HEAP_IMPL(NAME, T, LESS)                                                   \
    static void NAME##_push(T *h, int *n, T x) {                                   \
        int i = (*n)++;                                                            \
        while (i > 0) {                                                            \
            int p = (i - 1) >> 1;                                                  \
            if (!LESS(&x, &h[p])) break;                                           \
            h[i] = h[p];                                                           \
            i = p;                                                                 \
        }                                                                          \
        h[i] = x;                                                                  \
    }                                                                              \
    static T NAME##_pop(T *h, int *n) {                                            \
        T top = h[0], x = h[--(*n)];                                               \
        int i = 0;                                                                 \
        for (;;) {                                                                 \
            int c = 2 * i + 1;                                                     \
            if (c >= *n) break;                                                    \
            if (c + 1 < *n && LESS(&h[c + 1], &h[c])) c++;                         \
            if (!LESS(&h[c], &x)) break;                                           \
            h[i] = h[c];                                                           \
            i = c;                                                                 \
        }                                                                          \
        if (*n > 0) h[i] = x;                                                      \
        return top;                                                                \
    }

HEAP_IMPL(ev, ev_t, ev_less)
HEAP_IMPL(rq, rq_t, rq_less)

typedef struct {
    int n, d;
    const double *cost;      /* [n] by gid */
    const int32_t *rank;     /* [n] topo rank of gid */
    const int32_t *indeg;    /* [n] distinct predecessor groups */
    const int32_t *eoff;     /* [n+1] CSR by src gid */
    const int32_t *edst;     /* [E] dst gid, each row sorted by rank[dst] */
    const int64_t *ebytes;   /* [E] */
    const int64_t *resident; /* [n] param_bytes + out_bytes */
    const double *rate;      /* [d] */
    const double *bw;        /* [d*d] */
    const int64_t *mem;      /* [d] */
} oracle_graph;

/* One placement.  Returns 0, or 1 on an out-of-range device id. */
static int simulate_one(const oracle_graph *g, const uint8_t *pl, double *makespan, double *busy,
                        double *transfer, int64_t *peak, uint8_t *feasible, int32_t *order,
                        void *scratch) {
    const int n = g->n, d = g->d;
    for (int i = 0; i < n; i++)
        if (pl[i] >= d) return 1;
    char *p = (char *)scratch;
    int *pending = (int *)p;            p += sizeof(int) * n;
    double *finish = (double *)p;       p += sizeof(double) * n;
    ev_t *evh = (ev_t *)p;              p += sizeof(ev_t) * (n + g->eoff[n] + 1);
    rq_t *rqh = (rq_t *)p;              p += sizeof(rq_t) * (size_t)n * d;
    int *rqn = (int *)p;                p += sizeof(int) * d;
    int *idle = (int *)p;               p += sizeof(int) * d;
    double *link = (double *)p;         p += sizeof(double) * d * d;
    int nev = 0, nord = 0;
    for (int i = 0; i < n; i++) { pending[i] = g->indeg[i]; finish[i] = 0.0; }
    for (int j = 0; j < d; j++) { rqn[j] = 0; idle[j] = 1; busy[j] = 0.0; transfer[j] = 0.0; }
    for (int j = 0; j < d * d; j++) link[j] = 0.0;

#define START_NEXT(dev, now)                                                        \
    do {                                                                            \
        int dv_ = (dev);                                                            \
        if (idle[dv_] && rqn[dv_] > 0) {                                            \
            rq_t r_ = rq_pop(rqh + (size_t)dv_ * n, &rqn[dv_]);                     \
            if (order) order[nord++] = r_.gid;                                      \
            idle[dv_] = 0;                                                          \
            double dur_ = g->cost[r_.gid] / g->rate[pl[r_.gid]];                    \
            busy[dv_] += dur_;                                                      \
            ev_t e_ = {(now) + dur_, 0, g->rank[r_.gid], r_.gid};                   \
            ev_push(evh, &nev, e_);                                                 \
        }                                                                           \
    } while (0)

    for (int gi = 0; gi < n; gi++) {
        if (pending[gi] == 0) {
            rq_t r = {0.0, g->rank[gi], gi};
            rq_push(rqh + (size_t)pl[gi] * n, &rqn[pl[gi]], r);
        }
    }
    for (int dv = 0; dv < d; dv++) START_NEXT(dv, 0.0);

    while (nev > 0) {
        ev_t e = ev_pop(evh, &nev);
        if (e.kind == 0) {
            finish[e.gid] = e.t;
            int dev = pl[e.gid];
            idle[dev] = 1;
            for (int k = g->eoff[e.gid]; k < g->eoff[e.gid + 1]; k++) {
                int dst = g->edst[k];
                int ddev = pl[dst];
                double arrive;
                if (ddev == dev || g->ebytes[k] == 0) {
                    arrive = e.t;
                } else {
                    double lf = link[dev * d + ddev];
                    double begin = e.t > lf ? e.t : lf; /* Python max(t, lf): t wins ties */
                    double dur = (double)g->ebytes[k] / g->bw[dev * d + ddev];
                    link[dev * d + ddev] = begin + dur;
                    transfer[dev] += dur;
                    arrive = begin + dur;
                }
                ev_t a = {arrive, 1, g->rank[dst], dst};
                ev_push(evh, &nev, a);
            }
            START_NEXT(dev, e.t);
        } else {
            if (--pending[e.gid] == 0) {
                int dev = pl[e.gid];
                rq_t r = {e.t, g->rank[e.gid], e.gid};
                rq_push(rqh + (size_t)dev * n, &rqn[dev], r);
                START_NEXT(dev, e.t);
            }
        }
    }
#undef START_NEXT
    double mk = 0.0;
    for (int i = 0; i < n; i++)
        if (i == 0 || finish[i] > mk) mk = finish[i];
    *makespan = n ? mk : 0.0;
    for (int j = 0; j < d; j++) peak[j] = 0;
    for (int i = 0; i < n; i++) peak[pl[i]] += g->resident[i];
    int ok = 1;
    for (int j = 0; j < d; j++)
        if (peak[j] > g->mem[j]) ok = 0;
    *feasible = (uint8_t)ok;
    return 0;
}

static size_t scratch_bytes(int n, int d, int e) {
    return sizeof(int) * n + sizeof(double) * n + sizeof(ev_t) * (size_t)(n + e + 1) +
           sizeof(rq_t) * (size_t)n * d + sizeof(int) * 2 * d + sizeof(double) * d * d + 64;
}

typedef struct {
    const oracle_graph *g;
    const uint8_t *pl;
    double *makespan, *busy, *transfer;
    int64_t *peak;
    uint8_t *feasible;
    int32_t *order;
    int K, tid, nthreads, bad;
    size_t sb;
} worker_t;

static void *worker(void *arg) {
    worker_t *w = (worker_t *)arg;
    const oracle_graph *g = w->g;
    int n = g->n, d = g->d;
    void *scratch = malloc(w->sb);
    w->bad = -1;
    for (int k = w->tid; k < w->K; k += w->nthreads) {
        int rc = simulate_one(g, w->pl + (size_t)k * n, w->makespan + k, w->busy + (size_t)k * d,
                              w->transfer + (size_t)k * d, w->peak + (size_t)k * d, w->feasible + k,
                              w->order ? w->order + (size_t)k * n : NULL, scratch);
        if (rc && w->bad < 0) w->bad = k;
    }
    free(scratch);
    return NULL;
}

/* K placements ([K*n] by gid).  order may be NULL.  nthreads>1 uses pthreads
 * (placements are independent; results do not depend on the thread count).
 * Returns 0 ok, 1 bad device id (lowest offending placement index in *bad). */
int oracle_simulate_batch(int n, const double *cost, const int32_t *rank, const int32_t *indeg,
                          const int32_t *eoff, const int32_t *edst, const int64_t *ebytes,
                          const int64_t *resident, int d, const double *rate, const double *bw,
                          const int64_t *mem, int K, const uint8_t *placements, double *makespan,
                          double *busy, double *transfer, int64_t *peak, uint8_t *feasible,
                          int32_t *order, int nthreads, int *bad) {
    oracle_graph g = {n, d, cost, rank, indeg, eoff, edst, ebytes, resident, rate, bw, mem};
    if (nthreads < 1) nthreads = 1;
    if (nthreads > K) nthreads = K > 0 ? K : 1;
    worker_t *ws = (worker_t *)calloc((size_t)nthreads, sizeof(worker_t));
    pthread_t *th = (pthread_t *)calloc((size_t)nthreads, sizeof(pthread_t));
    for (int i = 0; i < nthreads; i++) {
        worker_t w = {&g, placements, makespan, busy, transfer, peak, feasible, order,
                      K, i, nthreads, -1, scratch_bytes(n, d, eoff[n])};
        ws[i] = w;
        if (nthreads == 1) worker(&ws[i]);
        else pthread_create(&th[i], NULL, worker, &ws[i]);
    }
    if (nthreads > 1)
        for (int i = 0; i < nthreads; i++) pthread_join(th[i], NULL);
    *bad = -1;
    for (int i = 0; i < nthreads; i++)
        if (ws[i].bad >= 0 && (*bad < 0 || ws[i].bad < *bad)) *bad = ws[i].bad;
    free(ws);
    free(th);
    return *bad >= 0;
}
