"""TEST INFRASTRUCTURE ONLY — the reference's own code, timed on the host cores.

bench.py's reference arm (``--impl reference``) and its ``cpu_baseline`` leg run
the UNMODIFIED reference package installed by ``oracle/make_ref.sh`` into
``oracle/_ref`` (``devplace``, pure Python + numpy).  Nothing here is a
restatement: every per-placement operation is a call into the reference.

* **Step** (R1 on all cores) — one REINFORCE update of ``run_controller``
  (``pkg/trainer.py:271-308``) for K placements: the reference's
  ``forward_sample`` (``pkg/policy.py:317-326``), ``measure`` through the
  trainer's ``_measure_one`` (``pkg/trainer.py:244-253``), ``reward_of``
  (``:66-72``) and ``grad_log_prob(cache=...)`` (``pkg/policy.py:351-409``) run
  in a persistent ``fork`` pool (one process per host core, BLAS pinned to one
  thread, pool created outside the timed region); sample k of the update
  consumes draws k*T.. of the controller stream exactly as the sequential loop
  does.  The parent applies the reference's best / success-only / baseline
  logic, ``BaselineState.update`` and ``ParameterStore.apply`` (Adam).  The
  only regrouping is the advantage-weighted gradient sum
  (``pkg/trainer.py:149-152``), formed as per-worker partial sums.
* **R1 single process** — the reference's ``train()`` as shipped (one process,
  its thread pool), ``LogRow.wall_ms`` of the second update.
* **R2 scorer only** — the reference's ``simulate`` (``pkg/simulator.py:122-194``)
  over a batch of random placements on a ``fork`` pool, chunked.
"""

from __future__ import annotations

import math
import multiprocessing as mp
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_DIR = os.path.join(HERE, "_ref")
ROOT = os.path.dirname(HERE)

_W: dict = {}  # per-process state (built once per worker)


def available() -> bool:
    return os.path.exists(os.path.join(REF_DIR, "devplace", "__init__.py"))


def load_reference():
    """Import the installed reference package (``devplace``)."""
    if not available():
        raise RuntimeError(f"reference not installed at {REF_DIR} (oracle/make_ref.sh)")
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    import devplace

    if not os.path.abspath(devplace.__file__).startswith(REF_DIR):
        raise RuntimeError(f"'devplace' resolves to {devplace.__file__}, not the reference install")
    return devplace


def _pin_blas():
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    os.environ["OMP_NUM_THREADS"] = "1"
    os.environ["MKL_NUM_THREADS"] = "1"
    try:
        from threadpoolctl import threadpool_limits

        threadpool_limits(1)
    except Exception:  # pragma: no cover
        pass


def reference_instance(cfg_path):
    """Rebuild a config instance (tests/golden/cfg_*.npz) with the reference's
    own constructors (``pkg/graph.py:34-190``, ``pkg/simulator.py:45-81``)."""
    ref = load_reference()
    from devplace.graph import ComputationGraph, Edge, GroupedGraph, Operation
    from devplace.simulator import Device, DeviceTopology

    with np.load(cfg_path, allow_pickle=False) as a:
        a = {k: a[k] for k in a.files}
    types = [str(t) for t in a["types"]]
    sp, dims = a["shape_ptr"], a["shape_dims"]
    ops = [Operation(i, f"op{i}", types[int(a["op_type"][i])], float(a["op_cost"][i]),
                     tuple(int(x) for x in dims[sp[i]:sp[i + 1]]), int(a["op_param"][i]))
           for i in range(len(a["op_type"]))]
    edges = [Edge(int(s), int(d), int(b)) for s, d, b in zip(a["edge_src"], a["edge_dst"], a["edge_bytes"])]
    pp, po = a["part_ptr"], a["part_ops"]
    parts = [tuple(int(x) for x in po[pp[i]:pp[i + 1]]) for i in range(len(pp) - 1)]
    gg = GroupedGraph(ComputationGraph(ops, edges), parts)
    devs = [Device(i, "gpu" if int(k) else "cpu", float(r), int(m))
            for i, (k, r, m) in enumerate(zip(a["dev_kind"], a["dev_rate"], a["dev_mem"]))]
    topo = DeviceTopology(devs, [[float(x) for x in row] for row in a["bw"]])
    return ref, gg, topo


def _task(cfg_path, seed, k):
    ref, gg, topo = reference_instance(cfg_path)
    tr = ref.trainer
    config = tr.TrainerConfig(k=k, total_updates=1, seed=seed)
    template = tr.policy_template(gg, topo, config)
    feats = ref.policy.GroupFeatures.from_grouped(gg, template.spec)
    spec = tr.RewardSpec(tr.suggest_failing_signal(gg, topo))
    tr.validate_failing_signal(spec, gg, topo)
    return ref, tr._TrainTask(gg, topo, feats, template, spec, config)


def _worker_init(cfg_path, seed, k):
    _pin_blas()
    ref, task = _task(cfg_path, seed, k)
    _W.update(ref=ref, task=task)


def _worker_chunk(args):
    """Samples k0..k1-1 of one update: the reference's per-placement work."""
    flat, state, inc, k0, k1, b, noise_seeds = args
    ref, task = _W["ref"], _W["task"]
    tr, pol = ref.trainer, ref.policy
    params = task.template.with_flat(flat)
    rng = np.random.Generator(np.random.PCG64())
    rng.bit_generator.state = {"bit_generator": "PCG64", "state": {"state": state, "inc": inc},
                               "has_uint32": 0, "uinteger": 0}
    rng.bit_generator.advance(k0 * len(task.feats))
    P = params.flat_size
    s_all, s_feas = np.zeros(P), np.zeros(P)
    out = []
    for i, k in enumerate(range(k0, k1)):
        s = pol.forward_sample(params, task.feats, rng)
        m = tr._measure_one(task, s.placement, noise_seeds[i])
        r = tr.reward_of(m, task.reward_spec)
        ok = m != ref.simulator.INFEASIBLE
        g = pol.grad_log_prob(params, task.feats, s.placement, cache=s.cache)
        s_all += (r - b) * g
        if ok:
            s_feas += (r - b) * g
        out.append((s.placement, s.log_prob, m, r, ok))
    return out, s_all, s_feas


class RefStepper:
    """Persistent process pool running full reference REINFORCE updates."""

    def __init__(self, cfg_path, k, seed=0, workers=None):
        _pin_blas()
        self.workers = workers or len(os.sched_getaffinity(0))
        self.k = k
        self.ref, self.task = _task(cfg_path, seed, k)
        tr = self.ref.trainer
        cfg = self.task.config
        self.store = tr.ParameterStore(self.task.template.to_flat(), learning_rate=cfg.learning_rate,
                                       beta1=cfg.adam_beta1, beta2=cfg.adam_beta2, epsilon=cfg.adam_epsilon)
        s_seq, n_seq = np.random.SeedSequence(seed).spawn(1)[0].spawn(2)
        self.rng = np.random.default_rng(s_seq)
        self.noise_rng = np.random.default_rng(n_seq)
        self.baseline = tr.BaselineState(value=self.task.reward_spec.failing_signal, decay=cfg.baseline_decay,
                                         initialized_from_failing_signal=True)
        self.best_r, self.update = math.inf, 0
        self.pool = mp.get_context("fork").Pool(self.workers, initializer=_worker_init,
                                                initargs=(cfg_path, seed, k))
        self.T = len(self.task.feats)

    def close(self):
        self.pool.close()
        self.pool.join()

    def step(self):
        """One update (``pkg/trainer.py:271-308``); returns (placements done, rows)."""
        tr, cfg, K = self.ref.trainer, self.task.config, self.k
        flat, _ = self.store.snapshot()
        st = self.rng.bit_generator.state["state"]
        noise = [int(self.noise_rng.integers(1 << 62)) for _ in range(K)]
        per = -(-K // self.workers)
        b = self.baseline.value
        jobs = [(flat, st["state"], st["inc"], k0, min(K, k0 + per), b, noise[k0:k0 + per])
                for k0 in range(0, K, per)]
        res = self.pool.map(_worker_chunk, jobs)
        self.rng.bit_generator.advance(K * self.T)
        rows = [r for chunk, _, _ in res for r in chunk]
        rewards = [r[3] for r in rows]
        feasible = [r[4] for r in rows]
        for (pl, _lp, _m, r, ok) in rows:
            if ok and r < self.best_r:
                self.best_r = r
        if self.update < cfg.success_only_after:
            used = list(range(K))
            g = sum(s for _, s, _ in res)
        else:
            used = [i for i in range(K) if feasible[i]]
            g = sum(s for _, _, s in res)
        if used:
            g = g / len(used)
            self.baseline.update(float(np.mean([rewards[i] for i in used])))
            self.store.apply(g)
        self.update += 1
        return K, float(np.mean(rewards))


def time_steps(cfg_path, k, steps, warmup, workers=None):
    """Warm-up + timed reference updates on all cores; returns a dict."""
    rs = RefStepper(cfg_path, k, workers=workers)
    try:
        for _ in range(warmup):
            rs.step()
        t0 = time.perf_counter()
        n = 0
        for _ in range(steps):
            n += rs.step()[0]
        dt = time.perf_counter() - t0
    finally:
        rs.close()
    return {"placements": n, "seconds": dt, "rate": n / dt if dt > 0 else None, "workers": rs.workers}


def single_process_rate(cfg_path, k=16, seed=0):
    """R1 as shipped: the reference ``train()`` in this one process (BLAS one
    thread), K=k, 2 updates; placements/s of the second (steady) update."""
    _pin_blas()
    ref, gg, topo = reference_instance(cfg_path)
    res = ref.trainer.train(gg, topo, ref.trainer.TrainerConfig(k=k, total_updates=2, seed=seed))
    wall = res.log[-1].wall_ms
    return {"rate": k / (wall * 1e-3), "k": k, "update_ms": wall}


def _sim_init(cfg_path):
    _pin_blas()
    ref, gg, topo = reference_instance(cfg_path)
    _W.update(ref=ref, gg=gg, topo=topo)


def _sim_chunk(placements):
    ref, gg, topo = _W["ref"], _W["gg"], _W["topo"]
    return [ref.simulator.simulate(gg, topo, [int(x) for x in p]).makespan_seconds for p in placements]


def scorer_rate(cfg_path, n=4096, workers=None, seed=1):
    """R2: the reference's simulate over n random placements on a fork pool."""
    workers = workers or len(os.sched_getaffinity(0))
    ref, gg, topo = reference_instance(cfg_path)
    pl = np.random.default_rng(seed).integers(0, topo.num_devices, (n, gg.num_groups))
    chunks = [c for c in np.array_split(pl, workers) if len(c)]
    with mp.get_context("fork").Pool(workers, initializer=_sim_init, initargs=(cfg_path,)) as pool:
        pool.map(_sim_chunk, [c[:2] for c in chunks])  # warm
        t0 = time.perf_counter()
        out = pool.map(_sim_chunk, chunks)
        dt = time.perf_counter() - t0
    return {"rate": n / dt, "placements": n, "seconds": dt, "workers": workers,
            "makespans": np.concatenate([np.asarray(o) for o in out])}
