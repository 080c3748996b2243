"""SPEC acceptance #4 (RL optimality on enumerable instances,
/root/reference/SPEC.md:492) on the device trainer: 10 seeded runs of train()
(1 controller, K=4, <= 1000 updates, success_only_after=50) on a generated
8-group / 2-device graph (256 placements) must return a placement whose
makespan equals brute_force's optimum (pkg/baselines.py:254-273) in >= 9/10
runs.  Plus the failing-signal property (#6): when every single-device
placement is memory-infeasible, training still returns a feasible placement."""

import numpy as np
import pytest

import paper_1706_04972_b200 as dp
from paper_1706_04972_b200 import graph as G
from paper_1706_04972_b200.simulator import Device, DeviceTopology

pytestmark = pytest.mark.gpu


def fork_join_instance(mem=1 << 40):
    """8 ops: a source, six independent branches of unequal cost, a sink.
    Balancing the branches over both devices beats either device alone."""
    costs = [0.5, 3.0, 2.0, 2.5, 1.5, 1.0, 3.5, 0.5]
    ops = [G.Operation(i, f"op{i}", "matmul" if 0 < i < 7 else "io", c, (256,), 1 << 20) for i, c in enumerate(costs)]
    edges = [G.Edge(0, b, 64) for b in range(1, 7)] + [G.Edge(b, 7, 64) for b in range(1, 7)]
    gg = G.singleton_groups(G.ComputationGraph(ops, edges))
    topo = DeviceTopology([Device(0, "gpu", 1.0, mem), Device(1, "gpu", 1.0, mem)],
                          [[0.0, 1024.0], [1024.0, 0.0]])
    return gg, topo


def test_rl_reaches_brute_force_optimum():
    gg, topo = fork_join_instance()
    best_pl, best_ms = dp.brute_force(gg, topo)
    single = min(dp.simulate(gg, topo, [d] * gg.num_groups).makespan_seconds for d in range(2))
    assert best_ms < single  # the optimum uses both devices
    hits = 0
    for seed in range(10):
        cfg = dp.TrainerConfig(k=4, total_updates=1000, success_only_after=50, seed=seed)
        res = dp.train(gg, topo, cfg)
        assert res.found_feasible
        ms = dp.simulate(gg, topo, res.best_placement).makespan_seconds
        assert ms >= best_ms
        hits += ms == best_ms
    assert hits >= 9, hits


def test_failing_signal_returns_feasible_placement():
    """Every op holds 1 MiB of parameters; 5 MiB per device makes both
    single-device placements infeasible while balanced splits fit."""
    gg, topo = fork_join_instance(mem=5 << 20)
    for d in range(2):
        assert not dp.simulate(gg, topo, [d] * gg.num_groups).feasible
    res = dp.train(gg, topo, dp.TrainerConfig(k=4, total_updates=300, success_only_after=50, seed=3))
    assert res.found_feasible and res.best_report.feasible
    # after success_only_after, updates only ever consumed feasible samples
    for row in res.log:
        if row.update_index >= 50:
            assert row.n_used == row.n_feasible
