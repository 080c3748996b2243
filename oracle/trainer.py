"""TEST INFRASTRUCTURE ONLY — restatement of one single-controller REINFORCE run.

Follows /root/reference/pkg/src/devplace/trainer.py:
* failing signal / validation  trainer.py:46-63
* reward_of                    trainer.py:66-72
* baseline moving average      trainer.py:75-84
* Adam (ParameterStore.apply)  trainer.py:113-131
* reinforce_update             trainer.py:138-154
* one controller round         trainer.py:256-309 (RNG streams trainer.py:260-262, 362-363)
* LogRow CSV                   trainer.py:187-224

Uses oracle.policy for sampling/gradients and oracle.sim for scoring.  Also
exposes ``cpu_step_rate`` — the bounded CPU-baseline sample bench.py times.
"""

from __future__ import annotations

import math
import os
import time

import numpy as np

from . import policy as opol
from .sim import OracleGraph

INF = math.inf


def failing_signal(gg, topo) -> float:
    slowest = min(d.compute_rate for d in topo.devices)
    return 2.0 * math.sqrt(gg.total_compute_cost() / slowest)


def reward(m: float, failing: float) -> float:
    if m == INF:
        return failing
    if not math.isfinite(m) or m <= 0:
        raise ValueError(f"measurement must be positive and finite, got {m}")
    return math.sqrt(m)


class Adam:
    def __init__(self, flat, lr=1e-3, b1=0.9, b2=0.999, eps=1e-8):
        self.x = np.array(flat, np.float64)
        self.m = np.zeros_like(self.x)
        self.v = np.zeros_like(self.x)
        self.t = 0
        self.lr, self.b1, self.b2, self.eps = lr, b1, b2, eps
        self.version = 0
        self.rejected = 0

    def apply(self, g) -> int:
        g = np.asarray(g, np.float64)
        if g.shape != self.x.shape:
            raise ValueError(f"gradient length {g.shape} != parameter length {self.x.shape}")
        if not np.isfinite(g).all():
            self.rejected += 1
            return self.version
        self.t += 1
        self.m = self.b1 * self.m + (1.0 - self.b1) * g
        self.v = self.b2 * self.v + (1.0 - self.b2) * g * g
        mh = self.m / (1.0 - self.b1 ** self.t)
        vh = self.v / (1.0 - self.b2 ** self.t)
        self.x -= self.lr * mh / (np.sqrt(vh) + self.eps)
        self.version += 1
        return self.version


def dims_for(gg, topo, cfg) -> opol.Dims:
    return opol.Dims(len(opol.vocab_of(gg)) + 1, topo.num_devices, cfg.get("hidden", 64),
                     cfg.get("dev_dim", 16), cfg.get("type_dim", 16), cfg.get("shape_slots", 8),
                     cfg.get("adjacency_slots", 64))


def run(gg, topo, cfg: dict, record=False):
    """Single-controller train(); cfg uses TrainerConfig field names."""
    K, U = cfg["k"], cfg["total_updates"]
    seed = cfg.get("seed", 0)
    dims = dims_for(gg, topo, cfg)
    feats = opol.features(gg, opol.vocab_of(gg), dims.shape_slots, dims.adj_slots)
    fail = cfg.get("failing_signal") or failing_signal(gg, topo)
    if not fail > math.sqrt(gg.total_compute_cost() / min(d.compute_rate for d in topo.devices)):
        raise ValueError("failing_signal does not exceed the slowest-single-device bound")
    store = Adam(opol.init_flat(dims, seed, cfg.get("init_scale", 0.1)), cfg.get("learning_rate", 1e-3),
                 cfg.get("adam_beta1", 0.9), cfg.get("adam_beta2", 0.999), cfg.get("adam_epsilon", 1e-8))
    s_seq, n_seq = np.random.SeedSequence(seed).spawn(1)[0].spawn(2)
    srng, nrng = np.random.default_rng(s_seq), np.random.default_rng(n_seq)
    base = fail
    decay = cfg.get("baseline_decay", 0.9)
    soa = cfg.get("success_only_after", 5000)
    og = OracleGraph(gg, topo)
    best_r, best_pl = INF, None
    rows, rec = [], {"placements": [], "logp": [], "measure": [], "grads": []}
    for upd in range(U):
        pol = opol.Policy(store.x.copy(), dims, feats)
        draws = [pol.sample(srng) for _ in range(K)]
        # noise seeds are drawn even with noise off (trainer.py:277)
        seeds = [int(nrng.integers(1 << 62)) for _ in range(K)]
        rep = og.simulate([s[0] for s in draws])
        sigma, steps = cfg.get("noise_sigma", 0.0), cfg.get("measure_steps", 10)
        meas = []
        for m, f, sd in zip(rep["makespan"], rep["feasible"], seeds):
            if steps < 2 or not f:  # measure() raises (-> INFEASIBLE) / infeasible
                meas.append(INF)
            elif sigma > 0.0:  # simulator.py:221-223
                fac = np.exp(sigma * np.random.default_rng(sd).standard_normal(steps))
                meas.append(float(np.mean(float(m) * fac[1:])))
            else:
                meas.append(float(m))
        rw = [reward(m, fail) for m in meas]
        ok = [m != INF for m in meas]
        for s, r, good in zip(draws, rw, ok):
            if good and r < best_r:
                best_r, best_pl = r, list(s[0])
        used = list(range(K)) if upd < soa else [i for i in range(K) if ok[i]]
        grad = None
        if used:
            b = base
            grad = np.zeros(dims.n_params)
            for i in used:
                grad += (rw[i] - b) * pol.grad(draws[i][0], draws[i][2])
            grad /= len(used)
            base = decay * base + (1.0 - decay) * float(np.mean([rw[i] for i in used]))
        ver = store.apply(grad) if grad is not None else store.version
        rows.append((upd, 0, ver, float(np.mean(rw)), base, best_r, sum(ok), len(used)))
        if record:
            rec["placements"].append([s[0] for s in draws])
            rec["logp"].append([s[1] for s in draws])
            rec["measure"].append(meas)
            rec["grads"].append(grad)
    return dict(rows=rows, final=store.x, best_placement=best_pl, best_r=best_r,
                versions=store.version, rejected=store.rejected, **rec)


def run_multi(gg, topo, cfg: dict):
    """C controllers sharing one store (pkg/trainer.py:365-378) under the
    deterministic round schedule the device runner uses: every round all
    controllers sample from the same store version, then apply in controller
    order.  (One of the reference's admissible asynchronous interleavings; with
    C == 1 it is exactly ``run``.)  Rows sorted by (controller, update)."""
    K, U, C = cfg["k"], cfg["total_updates"], cfg.get("controllers", 1)
    seed = cfg.get("seed", 0)
    dims = dims_for(gg, topo, cfg)
    feats = opol.features(gg, opol.vocab_of(gg), dims.shape_slots, dims.adj_slots)
    fail = cfg.get("failing_signal") or failing_signal(gg, topo)
    store = Adam(opol.init_flat(dims, seed, cfg.get("init_scale", 0.1)), cfg.get("learning_rate", 1e-3),
                 cfg.get("adam_beta1", 0.9), cfg.get("adam_beta2", 0.999), cfg.get("adam_epsilon", 1e-8))
    decay = cfg.get("baseline_decay", 0.9)
    soa = cfg.get("success_only_after", 5000)
    og = OracleGraph(gg, topo)
    ctl = []
    for cs in np.random.SeedSequence(seed).spawn(C):
        s_seq, n_seq = cs.spawn(2)
        ctl.append(dict(srng=np.random.default_rng(s_seq), nrng=np.random.default_rng(n_seq), base=fail,
                        best_r=INF, best_pl=None, rows=[]))
    for upd in range(U):
        snap = store.x.copy()
        grads = []
        for c in ctl:
            pol = opol.Policy(snap.copy(), dims, feats)
            draws = [pol.sample(c["srng"]) for _ in range(K)]
            for _ in range(K):
                c["nrng"].integers(1 << 62)
            rep = og.simulate([d[0] for d in draws])
            meas = [float(m) if f else INF for m, f in zip(rep["makespan"], rep["feasible"])]
            rw = [reward(m, fail) for m in meas]
            ok = [m != INF for m in meas]
            for d, r, good in zip(draws, rw, ok):
                if good and r < c["best_r"]:
                    c["best_r"], c["best_pl"] = r, list(d[0])
            used = list(range(K)) if upd < soa else [i for i in range(K) if ok[i]]
            grad = None
            if used:
                b = c["base"]
                grad = np.zeros(dims.n_params)
                for i in used:
                    grad += (rw[i] - b) * pol.grad(draws[i][0], draws[i][2])
                grad /= len(used)
                c["base"] = decay * b + (1.0 - decay) * float(np.mean([rw[i] for i in used]))
            grads.append((grad, float(np.mean(rw)), sum(ok), len(used)))
        for cid, (c, (grad, mr, nf, nu)) in enumerate(zip(ctl, grads)):
            ver = store.apply(grad) if grad is not None else store.version
            c["rows"].append((upd, cid, ver, mr, c["base"], c["best_r"], nf, nu))
    best = min(ctl, key=lambda c: c["best_r"])
    rows = [r for c in ctl for r in c["rows"]]
    return dict(rows=rows, final=store.x, best_placement=best["best_pl"], best_r=best["best_r"],
                versions=store.version, rejected=store.rejected)


def csv_of(rows) -> str:
    lines = ["update_index,controller_id,store_version,mean_R,baseline,best_R,n_feasible_of_K"]
    for (u, c, ver, mr, b, br, nf, _nu) in rows:
        lines.append(",".join([str(u), str(c), str(ver), repr(mr), repr(b), repr(br), str(nf)]))
    return "\n".join(lines) + "\n"


# ------------------------------------------------------------------ CPU baseline
def _sample_and_grad(args):
    flat, dims, feats, state, inc, first, count, og_args = args
    import numpy as _np

    gen = _np.random.Generator(_np.random.PCG64())
    gen.bit_generator.state = {"bit_generator": "PCG64", "state": {"state": state, "inc": inc},
                               "has_uint32": 0, "uinteger": 0}
    T = len(feats.order)
    gen.bit_generator.advance(first * T)
    pol = opol.Policy(flat, dims, feats)
    out = []
    for _ in range(count):
        pl, lp, tape = pol.sample(gen)
        out.append((pl, lp, pol.grad(pl, tape)))
    return out


def cpu_step_rate(gg, topo, k_sample: int, workers: int | None = None, seed: int = 0):
    """Time one REINFORCE update's worth of per-placement work (sample + score +
    gradient) for ``k_sample`` placements on ``workers`` processes.  Per-placement
    cost is independent of K, so placements/s extrapolates to any K."""
    import multiprocessing as mp

    workers = workers or len(os.sched_getaffinity(0))
    dims = dims_for(gg, topo, {})
    feats = opol.features(gg, opol.vocab_of(gg), dims.shape_slots, dims.adj_slots)
    flat = opol.init_flat(dims, seed)
    s_seq, _ = np.random.SeedSequence(seed).spawn(1)[0].spawn(2)
    st = np.random.default_rng(s_seq).bit_generator.state["state"]
    og = OracleGraph(gg, topo)
    chunks = [list(range(i, k_sample, workers)) for i in range(workers)]
    tasks = []
    per = -(-k_sample // workers)
    for w in range(workers):
        first = w * per
        cnt = max(0, min(per, k_sample - first))
        if cnt:
            tasks.append((flat, dims, feats, st["state"], st["inc"], first, cnt, None))
    del chunks
    t0 = time.perf_counter()
    if workers > 1:
        ctx = mp.get_context("fork")
        with ctx.Pool(len(tasks)) as pool:
            res = pool.map(_sample_and_grad, tasks)
    else:
        res = [_sample_and_grad(t) for t in tasks]
    flat_res = [r for chunk in res for r in chunk]
    rep = og.simulate([r[0] for r in flat_res], threads=workers)
    g = np.zeros(dims.n_params)
    for r, m in zip(flat_res, rep["makespan"]):
        g += (math.sqrt(m) - 1.0) * r[2]
    dt = time.perf_counter() - t0
    return dict(placements=len(flat_res), seconds=dt, rate=len(flat_res) / dt, workers=workers)
