"""Generate the golden fixtures under tests/golden/ by running the REFERENCE.

Run in the build container only (needs /root/reference):

    python tests/golden/make_golden.py

Everything here executes the unmodified reference package (`devplace`,
/root/reference/pkg/src) through its public API; nothing from this repo's
product code is used to compute expected values.  The outputs pin:

* cfg_*.npz          — config instances C1, C2, C3, C3tight, C5 (SURVEY.md §8(d),
                       Appendix E) in the compact form of
                       paper_1706_04972_b200/instances.py, plus the reference's
                       group-level arrays (costs, edges, topo) to pin the rebuild.
* sim_*.npz          — simulate() reports + dispatch orders (heapq shim,
                       SURVEY.md Appendix A.3) for seeded placements.
* sim_random.npz     — 300 tests/util.py random_instance cases (+ 100 with
                       zero-cost groups / zero-byte edges).
* policy_*.npz       — forward_sample placements/log-probs on the trainer's
                       sample stream, step_distributions, log_prob_of and
                       grad_log_prob at seed-0 init params.
* train_*.npz/.csv   — train() logs (byte-stable CSV), per-update sampled
                       placements / rewards / reinforce gradients, final params.
* meta.json          — numpy version, generation parameters.
"""

from __future__ import annotations

import heapq as _real_heapq
import json
import math
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, "/root/reference/pkg/tests")
sys.path.insert(0, REPO)

import devplace as ref  # noqa: E402  (the reference)
import devplace.simulator as ref_sim  # noqa: E402
import devplace.trainer as ref_trainer  # noqa: E402
import devplace.policy as ref_policy  # noqa: E402
import devplace.generators as ref_gen  # noqa: E402
import devplace.graph as ref_graph  # noqa: E402
import util as ref_util  # noqa: E402  (reference tests/util.py)

from paper_1706_04972_b200.instances import instance_arrays  # noqa: E402  (serializer only)


# --------------------------------------------------------------------------- configs
def G(spec):
    g = ref.generate(spec)
    return ref.coalesce_sole_consumers(ref.ComputationGraph(g.ops, g.edges))


def c3_topology(mem=1 << 30):
    devs = [ref.Device(i, "gpu", 10.0, mem) for i in range(4)]
    bw = [[0.0 if i == j else 65536.0 for j in range(4)] for i in range(4)]
    return ref.DeviceTopology(devs, bw)


def c5_instance():
    """SURVEY.md Appendix E, exact draw order."""
    rng = np.random.default_rng(0)
    types = ["matmul", "conv2d", "add", "relu", "concat", "softmax", "tanh", "mul"]
    ops, edges = [], []
    shapes = {}
    for g in range(2000):
        for j in range(10):
            oid = 10 * g + j
            shape = (int(rng.integers(1, 4097)),)
            typ = types[int(rng.integers(8))]
            cost = max(round(rng.uniform(0.01, 0.2) * 1024) / 1024, 1 / 1024)
            pb = int(rng.integers(0, 4096))
            ops.append(ref.Operation(oid, f"g{g}/op{j}", typ, cost, shape, pb))
            shapes[oid] = shape
            if j > 0:
                edges.append(ref.Edge(oid - 1, oid, 4 * shapes[oid - 1][0]))
    for g in range(1999):
        cand = np.arange(g + 1, min(g + 65, 2000))
        m = min(int(rng.integers(2, 5)), len(cand))
        for dst in sorted(rng.choice(cand, size=m, replace=False)):
            edges.append(ref.Edge(10 * g + 9, 10 * int(dst), int(rng.integers(1024, 65537))))
    gg = ref.GroupedGraph(ref.ComputationGraph(ops, edges),
                          [tuple(range(10 * g, 10 * g + 10)) for g in range(2000)])
    return gg, ref.default_topology(7)


def configs():
    out = {
        "C1": (G(ref.GeneratorSpec("rnnlm_grid", layers=2, steps=16, seed=0)), ref.default_topology(1), 8),
        "C2": (G(ref.GeneratorSpec("nmt_attention", layers=4, steps=11, seed=0)), ref.default_topology(4), 64),
        "C3": (G(ref.GeneratorSpec("inception_blocks", blocks=18, branches=4, seed=0)), c3_topology(), 256),
    }
    out["C3tight"] = (out["C3"][0], c3_topology(30 << 20), 256)
    gg5, t5 = c5_instance()
    out["C5"] = (gg5, t5, 4096)
    return out


def group_level(gg):
    return dict(
        g_cost=np.array([g.compute_cost for g in gg.groups]),
        g_param=np.array([g.param_bytes for g in gg.groups], np.int64),
        g_out=np.array([g.out_bytes for g in gg.groups], np.int64),
        ge_src=np.array([e.src for e in gg.group_edges], np.int32),
        ge_dst=np.array([e.dst for e in gg.group_edges], np.int32),
        ge_bytes=np.array([e.tensor_bytes for e in gg.group_edges], np.int64),
        topo=np.array(gg.topo, np.int32),
    )


# --------------------------------------------------------------------------- heapq shim
class _DispatchRecorder:
    """Module-global heapq replacement for devplace.simulator (Appendix A.3):
    ready-queue entries are 3-tuples, events 4-tuples."""

    def __init__(self):
        self.order = []

    def heappush(self, h, x):
        _real_heapq.heappush(h, x)

    def heappop(self, h):
        x = _real_heapq.heappop(h)
        if len(x) == 3:
            self.order.append(x[2])
        return x


def sim_with_order(gg, topo, placement):
    rec = _DispatchRecorder()
    ref_sim.heapq = rec
    try:
        rep = ref.simulate(gg, topo, placement)
    finally:
        ref_sim.heapq = _real_heapq
    return rep, rec.order


def sim_golden(gg, topo, placements):
    K, D = len(placements), topo.num_devices
    mk = np.zeros(K)
    busy = np.zeros((K, D))
    tr = np.zeros((K, D))
    peak = np.zeros((K, D), np.int64)
    feas = np.zeros(K, np.uint8)
    order = np.zeros((K, gg.num_groups), np.int32)
    for k, p in enumerate(placements):
        rep, o = sim_with_order(gg, topo, [int(x) for x in p])
        mk[k] = rep.makespan_seconds
        busy[k] = rep.per_device_busy_seconds
        tr[k] = rep.per_device_transfer_seconds
        peak[k] = rep.per_device_peak_bytes
        feas[k] = rep.feasible
        order[k] = o
    return dict(placements=np.asarray(placements, np.uint8), makespan=mk, busy=busy,
                transfer=tr, peak=peak, feasible=feas, order=order)


# --------------------------------------------------------------------------- random suite
def random_suite(n_plain=300, n_zero=100, seed=12345):
    """tests/util.py random_instance cases; the zero-cost variant rebuilds each
    instance with some zero costs and zero-byte edges (legal per pkg/graph.py:103-104)."""
    rng = np.random.default_rng(seed)
    cases = []
    for i in range(n_plain + n_zero):
        gg, topo = ref_util.random_instance(rng, max_groups=8, max_devices=3)
        if i >= n_plain:
            g = gg.graph
            ops = [ref.Operation(op.id, op.name, op.op_type,
                                 0.0 if rng.random() < 0.3 else op.compute_cost,
                                 op.output_shape, op.param_bytes) for op in g.ops]
            edges = [ref.Edge(e.src, e.dst, 0 if rng.random() < 0.3 else e.tensor_bytes)
                     for e in g.edges]
            gg = ref.singleton_groups(ref.ComputationGraph(ops, edges))
        pl = ref_util.random_placement(rng, gg, topo)
        rep, order = sim_with_order(gg, topo, pl)
        cases.append((gg, topo, pl, rep, order))
    # ragged concatenation
    out = {}
    inst = [instance_arrays(gg, topo) for gg, topo, *_ in cases]
    keys = list(inst[0].keys())
    for k in keys:
        if k == "types":
            continue
        arrs = [a[k] for a in inst]
        out[k + "__ptr"] = np.cumsum([0] + [a.size for a in arrs]).astype(np.int64)
        out[k + "__shape1"] = np.array([a.shape[1] if a.ndim == 2 else 0 for a in arrs], np.int64)
        out[k] = np.concatenate([a.ravel() for a in arrs]) if sum(a.size for a in arrs) else arrs[0].ravel()
    # type names per instance (tiny vocab) joined with '|'
    out["types_joined"] = np.array(["|".join(str(t) for t in a["types"]) for a in inst])
    out["placement"] = np.concatenate([np.asarray(c[2], np.uint8) for c in cases])
    out["placement__ptr"] = np.cumsum([0] + [len(c[2]) for c in cases]).astype(np.int64)
    out["makespan"] = np.array([c[3].makespan_seconds for c in cases])
    out["busy"] = np.concatenate([np.asarray(c[3].per_device_busy_seconds) for c in cases])
    out["transfer"] = np.concatenate([np.asarray(c[3].per_device_transfer_seconds) for c in cases])
    out["peak"] = np.concatenate([np.asarray(c[3].per_device_peak_bytes, np.int64) for c in cases])
    out["dev__ptr"] = np.cumsum([0] + [c[1].num_devices for c in cases]).astype(np.int64)
    out["feasible"] = np.array([c[3].feasible for c in cases], np.uint8)
    out["order"] = np.concatenate([np.asarray(c[4], np.int32) for c in cases])
    out["oracle_sim_makespan"] = np.array(
        [__import__("oracle_sim").oracle_makespan(c[0], c[1], c[2]) for c in cases])
    return out


# --------------------------------------------------------------------------- policy
def trainer_sample_rng(seed, controllers=1, cid=0):
    root = np.random.SeedSequence(seed)
    sample_seq, _ = root.spawn(controllers)[cid].spawn(2)
    return np.random.default_rng(sample_seq)


def policy_golden(gg, topo, n_samples, seed=0):
    cfg = ref.TrainerConfig(seed=seed)
    params = ref_trainer.policy_template(gg, topo, cfg)
    feats = ref.GroupFeatures.from_grouped(gg, params.spec)
    rng = trainer_sample_rng(seed)
    st = rng.bit_generator.state["state"]
    samples = [ref.forward_sample(params, feats, rng) for _ in range(n_samples)]
    pl = np.array([s.placement for s in samples], np.uint8)
    lp = np.array([s.log_prob for s in samples])
    s0 = samples[0]
    probs0 = ref.step_distributions(params, feats, s0.placement)
    grad0 = ref.grad_log_prob(params, feats, s0.placement, cache=s0.cache)
    other = np.random.default_rng(7).integers(0, topo.num_devices, gg.num_groups)
    other = [int(x) for x in other]
    lp_other = ref.log_prob_of(params, feats, other)
    grad_other = ref.grad_log_prob(params, feats, other)
    x = ref.embed_groups(params, feats)
    return dict(
        flat=params.to_flat(), placements=pl, log_probs=lp,
        pcg_state=np.array([st["state"] >> 64, st["state"] & ((1 << 64) - 1),
                            st["inc"] >> 64, st["inc"] & ((1 << 64) - 1)], np.uint64),
        probs0=probs0, grad0=grad0, other=np.array(other, np.uint8), lp_other=np.float64(lp_other),
        grad_other=grad_other, inputs=x,
        vocab=np.array(sorted(params.spec.type_vocab, key=params.spec.type_vocab.get)),
    )


# --------------------------------------------------------------------------- trainer
def train_golden(gg, topo, cfg):
    rec = {"placements": [], "logp": [], "measure": [], "grads": [], "baseline_before": []}
    orig_fs = ref_policy.forward_sample
    orig_ru = ref_trainer.reinforce_update
    orig_me = ref.measure

    def fs(params, feats, rng):
        s = orig_fs(params, feats, rng)
        rec["placements"].append(list(s.placement))
        rec["logp"].append(s.log_prob)
        return s

    def ru(params, feats, samples, rewards, baseline):
        rec["baseline_before"].append(baseline.value)
        g = orig_ru(params, feats, samples, rewards, baseline)
        rec["grads"].append(np.full(params.flat_size, np.nan) if g is None else g)
        return g

    ref_policy.forward_sample, ref_trainer.reinforce_update = fs, ru
    try:
        res = ref.train(gg, topo, cfg)
    finally:
        ref_policy.forward_sample, ref_trainer.reinforce_update = orig_fs, orig_ru
    U, K = cfg.total_updates, cfg.k
    # measure() runs on worker threads (completion order), so re-derive per k
    # (the simulator is pure; noise is off in these runs).
    rec["measure"] = [orig_me(gg, topo, p) for p in rec["placements"]]
    csv = ref.log_to_csv(res.log, include_wall=False)
    out = dict(
        placements=np.array(rec["placements"], np.uint8).reshape(U, K, -1),
        logp=np.array(rec["logp"]).reshape(U, K),
        measure=np.array(rec["measure"]).reshape(U, K),
        grads=np.array(rec["grads"]),
        baseline_before=np.array(rec["baseline_before"]),
        final_params=res.final_params,
        best_placement=np.array(res.best_placement if res.best_placement else [], np.uint8),
        best_makespan=np.float64(res.best_makespan if res.best_makespan is not None else np.nan),
        store_versions=np.int64(res.store_versions),
        rejected=np.int64(res.rejected_updates),
        cfg=np.array(json.dumps(cfg.__dict__)),
        csv=np.array(csv),
    )
    return out, csv


NOISE_RUNS = {
    # f2: lognormal measurement noise on (pkg/trainer.py:244-253, simulator.py:205-223)
    "C1noise": ("C1", dict(k=8, total_updates=3, seed=3, noise_sigma=0.25)),
    "C3noise": ("C3tight", dict(k=8, total_updates=3, seed=4, noise_sigma=0.5, success_only_after=1,
                                measure_steps=5)),
}


def baselines_golden(n=14, seed=777):
    """f3: reference brute_force / place_random_search on small instances
    (pkg/baselines.py:227-273), some memory-tight, plus random search on C1."""
    rng = np.random.default_rng(seed)
    out = {}
    for i in range(n):
        gg, topo = ref_util.random_instance(rng, max_groups=9, max_devices=3)
        if i % 3 == 2:  # memory-tight: some (or all) placements infeasible
            foot = sum(g.param_bytes + g.out_bytes for g in gg.groups)
            mem = int(foot * (0.35 if i % 2 else 0.05)) + 1
            topo = ref.DeviceTopology([ref.Device(d.id, d.kind, d.compute_rate, mem) for d in topo.devices],
                                      topo.bandwidth)
        for k, v in instance_arrays(gg, topo).items():
            out[f"i{i}_{k}"] = v
        try:
            pl, mk = ref.brute_force(gg, topo)
            out[f"i{i}_bf_placement"] = np.array(pl, np.uint8)
            out[f"i{i}_bf_makespan"] = np.float64(mk)
        except ref.NoFeasiblePlacement:
            out[f"i{i}_bf_placement"] = np.zeros(0, np.uint8)
            out[f"i{i}_bf_makespan"] = np.float64(np.nan)
        rs = ref.place_random_search(gg, topo, budget=5 + 3 * i, seed=i)
        out[f"i{i}_rs_budget"] = np.int64(5 + 3 * i)
        out[f"i{i}_rs_placement"] = np.array(rs if rs is not None else [], np.uint8)
    out["n"] = np.int64(n)
    gg, topo, _ = configs()["C1"]
    rs = ref.place_random_search(gg, topo, budget=300, seed=11)
    out["c1_rs_placement"] = np.array(rs, np.uint8)
    return out


def main_noise():
    cfgs = configs()
    for name, (base, kw) in NOISE_RUNS.items():
        gg, topo, _ = cfgs[base]
        out, csv = train_golden(gg, topo, ref.TrainerConfig(**kw))
        np.savez_compressed(os.path.join(HERE, f"train_{name}.npz"), **out)
        with open(os.path.join(HERE, f"train_{name}.csv"), "w") as fh:
            fh.write(csv)
        print("train", name, flush=True)


def main():
    t0 = time.time()
    cfgs = configs()
    meta = {"numpy": np.__version__, "generated_by": "tests/golden/make_golden.py",
            "reference": "/root/reference/pkg/src/devplace"}
    for name, (gg, topo, K) in cfgs.items():
        np.savez_compressed(os.path.join(HERE, f"cfg_{name}.npz"),
                            **instance_arrays(gg, topo), **group_level(gg), K=np.int64(K))
        print(name, "N", gg.num_groups, "E", len(gg.group_edges), "D", topo.num_devices, flush=True)
    # simulator goldens
    for name, (gg, topo, K) in cfgs.items():
        n = 4 if name == "C5" else 16
        pl = np.random.default_rng(1).integers(0, topo.num_devices, (n, gg.num_groups))
        np.savez_compressed(os.path.join(HERE, f"sim_{name}.npz"), **sim_golden(gg, topo, pl))
    print("sim goldens", time.time() - t0, flush=True)
    np.savez_compressed(os.path.join(HERE, "sim_random.npz"), **random_suite())
    print("random suite", time.time() - t0, flush=True)
    # policy goldens
    for name, n in (("C1", 4), ("C2", 2), ("C3", 2)):
        gg, topo, _ = cfgs[name]
        np.savez_compressed(os.path.join(HERE, f"policy_{name}.npz"), **policy_golden(gg, topo, n))
    print("policy goldens", time.time() - t0, flush=True)
    # trainer goldens
    runs = {
        "C1": ref.TrainerConfig(k=8, total_updates=3, seed=0),
        "C3tight": ref.TrainerConfig(k=16, total_updates=4, seed=0, success_only_after=2),
        "C2": ref.TrainerConfig(k=4, total_updates=2, seed=1),
    }
    for name, cfg in runs.items():
        gg, topo, _ = cfgs[name]
        out, csv = train_golden(gg, topo, cfg)
        np.savez_compressed(os.path.join(HERE, f"train_{name}.npz"), **out)
        with open(os.path.join(HERE, f"train_{name}.csv"), "w") as fh:
            fh.write(csv)
        print("train", name, time.time() - t0, flush=True)
    with open(os.path.join(HERE, "meta.json"), "w") as fh:
        json.dump(meta, fh, indent=1)
        fh.write("\n")


INGEST_SPECS = {
    "rnnlm_L2S20": dict(family="rnnlm_grid", layers=2, steps=20, seed=0),
    "nmt_L4S40": dict(family="nmt_attention", layers=4, steps=40, seed=0),
}


def ingest_golden(spec):
    """f4: a paper-scale generator graph (8.8k ops for nmt L4 S40) whose manual
    groups are cyclic.  The acyclic split under test (graph.split_cyclic_groups)
    provides the INPUT partition; every expected value below is the reference's
    own GroupedGraph / coalescing / GroupFeatures on that input."""
    from paper_1706_04972_b200.graph import split_cyclic_groups  # input only

    g = ref_gen.generate(ref_gen.GeneratorSpec(**spec))
    try:
        ref.coalesce_sole_consumers(g)
        raise AssertionError("expected the shipped manual groups to be cyclic")
    except ref_graph.GraphError:
        pass
    fixed = split_cyclic_groups(g)
    gg = ref.coalesce_sole_consumers(fixed)          # reference coalescing + validation
    espec = ref_policy.EmbeddingSpec.build([gg])
    feats = ref_policy.GroupFeatures.from_grouped(gg, espec)
    types = sorted({op.op_type for op in g.ops})
    tix = {t: i for i, t in enumerate(types)}
    shape_ptr = np.zeros(len(g.ops) + 1, np.int64)
    dims = []
    for i, op in enumerate(g.ops):
        dims.extend(op.output_shape)
        shape_ptr[i + 1] = len(dims)
    man_ptr = np.cumsum([0] + [len(x) for x in g.manual_groups])
    split_ptr = np.cumsum([0] + [len(x) for x in fixed.manual_groups])
    part_ptr = np.cumsum([0] + [len(grp.members) for grp in gg.groups])
    tl = [np.asarray(x, np.int32) for x in feats.type_indices]
    adj_t, adj_s = np.nonzero(feats.adj_blocks)
    return dict(
        types=np.array(types), op_type=np.array([tix[op.op_type] for op in g.ops], np.int32),
        op_cost=np.array([op.compute_cost for op in g.ops], np.float64),
        op_param=np.array([op.param_bytes for op in g.ops], np.int64),
        shape_ptr=shape_ptr, shape_dims=np.array(dims, np.int64),
        op_name_grad=np.array(["/grad_" in op.name for op in g.ops]),
        edge_src=np.array([e.src for e in g.edges], np.int32), edge_dst=np.array([e.dst for e in g.edges], np.int32),
        edge_bytes=np.array([e.tensor_bytes for e in g.edges], np.int64),
        manual_ptr=man_ptr, manual_ops=np.concatenate([np.asarray(x, np.int32) for x in g.manual_groups]),
        split_ptr=split_ptr, split_ops=np.concatenate([np.asarray(x, np.int32) for x in fixed.manual_groups]),
        part_ptr=part_ptr, part_ops=np.concatenate([np.asarray(grp.members, np.int32) for grp in gg.groups]),
        group_cost=np.array([grp.compute_cost for grp in gg.groups]),
        group_param=np.array([grp.param_bytes for grp in gg.groups], np.int64),
        group_out_bytes=np.array([grp.out_bytes for grp in gg.groups], np.int64),
        ge_src=np.array([e.src for e in gg.group_edges], np.int32),
        ge_dst=np.array([e.dst for e in gg.group_edges], np.int32),
        ge_bytes=np.array([e.tensor_bytes for e in gg.group_edges], np.int64),
        topo=np.array(gg.topo, np.int32), vocab=np.array(sorted(espec.type_vocab, key=espec.type_vocab.get)),
        f_type_off=np.cumsum([0] + [len(x) for x in tl]), f_type_idx=np.concatenate(tl),
        f_shape=np.asarray(feats.shape_blocks), f_adj_t=adj_t.astype(np.int32), f_adj_s=adj_s.astype(np.int16),
    )


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "ingest":
        for name, spec in INGEST_SPECS.items():
            np.savez_compressed(os.path.join(HERE, f"ingest_{name}.npz"), **ingest_golden(spec))
            print("ingest", name)
        sys.exit(0)
    if len(sys.argv) > 1 and sys.argv[1] == "noise":
        main_noise()
    elif len(sys.argv) > 1 and sys.argv[1] == "baselines":
        np.savez_compressed(os.path.join(HERE, "baselines.npz"), **baselines_golden())
        print("baselines")
    else:
        main()
