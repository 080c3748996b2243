"""GPU parity of the fused REINFORCE update (epilogue + Adam kernels, csrc/train.cu)
and of the drop-in trainer API against the reference's own train() runs."""

import numpy as np
import pytest
import torch

from fixtures import cfg, train_golden, PARAM_RTOL
import paper_1706_04972_b200 as dp

pytestmark = pytest.mark.gpu


def _cfg(d):
    return dp.TrainerConfig(**d)


@pytest.mark.parametrize("name", ["C1", "C3tight", "C2"])
def test_train_log_and_params_match_reference(name):
    gg, topo, _, _ = cfg(name)
    g = train_golden(name)
    res = dp.train(gg, topo, _cfg(g["cfg"]))
    # byte-identical training log (placements, rewards, baselines, versions)
    assert dp.log_to_csv(res.log, include_wall=False) == g["csv"]
    if len(g["best_placement"]):
        assert res.best_placement == [int(x) for x in g["best_placement"]]
        assert res.best_makespan == float(g["best_makespan"])
    else:
        assert res.best_placement is None
    assert res.store_versions == int(g["store_versions"])
    assert res.rejected_updates == int(g["rejected"])
    rel = np.linalg.norm(res.final_params - g["final_params"]) / np.linalg.norm(g["final_params"])
    assert rel < PARAM_RTOL
    np.testing.assert_allclose(res.final_params, g["final_params"], rtol=1e-6, atol=1e-12)


def test_reinforce_update_dropin_matches_reference_gradient():
    gg, topo, _, _ = cfg("C1")
    g = train_golden("C1")
    c = _cfg(g["cfg"])
    params = dp.trainer.policy_template(gg, topo, c)
    feats = dp.GroupFeatures.from_grouped(gg, params.spec)
    fail = dp.suggest_failing_signal(gg, topo)
    spec = dp.RewardSpec(fail)
    pls = g["placements"][0]
    samples = [dp.SampledPlacement([int(x) for x in p], 0.0, None) for p in pls]
    rewards = [dp.reward_of(m, spec) for m in g["measure"][0]]
    b = dp.BaselineState(fail)
    grad = dp.reinforce_update(params, feats, samples, rewards, b)
    ref = g["grads"][0]
    assert np.linalg.norm(grad - ref) / np.linalg.norm(ref) < 1e-9
    assert b.value == float(g["baseline_before"][1])


def test_parameter_store_known_answers():
    s = dp.ParameterStore(np.ones(10))
    assert s.apply(np.zeros(10)) == 1
    assert np.array_equal(s.snapshot()[0], np.ones(10))  # zero gradient: parameters unchanged
    g = np.linspace(-1, 1, 10)
    s.apply(g)
    assert s.apply(np.full(10, np.nan)) == 2 and s.rejected == 1
    with pytest.raises(ValueError):
        s.apply(np.zeros(3))
    # numpy recurrence, two steps
    x, m, v = np.ones(10), np.zeros(10), np.zeros(10)
    for t, gg in ((1, np.zeros(10)), (2, g)):
        m = 0.9 * m + (1.0 - 0.9) * gg
        v = 0.999 * v + (1.0 - 0.999) * gg * gg
        x -= 1e-3 * (m / (1.0 - 0.9 ** t)) / (np.sqrt(v / (1.0 - 0.999 ** t)) + 1e-8)
    assert np.array_equal(s.snapshot()[0], x)


def test_train_is_deterministic_and_graph_replay_equals_eager():
    gg, topo, _, _ = cfg("C1")
    c = dp.TrainerConfig(k=8, total_updates=4, seed=3)
    a = dp.train(gg, topo, c)
    b = dp.train(gg, topo, c)
    assert dp.log_to_csv(a.log, False) == dp.log_to_csv(b.log, False)
    assert np.array_equal(a.final_params, b.final_params)
    # eager (no graph) controller produces the identical trace
    task = dp.trainer._make_task(gg, topo, c)
    store = dp.ParameterStore(task.template.to_flat(), max_steps=8)
    ctl = dp.trainer.DeviceController(task, store, np.random.SeedSequence(3).spawn(1)[0])
    ctl.run(4, use_graph=False)
    torch.cuda.synchronize()
    assert dp.log_to_csv(ctl.rows(), False) == dp.log_to_csv(a.log, False)
    assert np.array_equal(store.snapshot()[0], a.final_params)


@pytest.mark.parametrize("name,graph", [("C1noise", "C1"), ("C3noise", "C3tight")])
def test_train_with_measurement_noise_matches_reference(name, graph):
    """f2 on the device path: host-drawn factor table + dp_apply_measurement_noise."""
    gg, topo, _, _ = cfg(graph)
    g = train_golden(name)
    res = dp.train(gg, topo, _cfg(g["cfg"]))
    assert dp.log_to_csv(res.log, include_wall=False) == g["csv"]
    assert res.store_versions == int(g["store_versions"])
    rel = np.linalg.norm(res.final_params - g["final_params"]) / np.linalg.norm(g["final_params"])
    assert rel < PARAM_RTOL
    if len(g["best_placement"]):
        assert res.best_placement == [int(x) for x in g["best_placement"]]


@pytest.mark.parametrize("K", [300, 4096])
def test_epilogue_pairwise_mean_large_k(K):
    """mean_R over K > 128 rewards follows numpy's recursive pairwise sum
    (restated iteratively on device) — byte-equal to np.mean."""
    import math

    gg, topo, _, _ = cfg("C1")
    c = dp.TrainerConfig(k=K, total_updates=1, seed=2)
    task = dp.trainer._make_task(gg, topo, c)
    store = dp.ParameterStore(task.template.to_flat(), max_steps=4)
    ctl = dp.trainer.DeviceController(task, store, np.random.SeedSequence(2).spawn(1)[0], 0)
    ctl.run(1, use_graph=False)
    torch.cuda.synchronize()
    row = ctl.rows()[0]
    out = ctl.dg.simulate(ctl.choice, by_rank=True)
    mk, fe = out["makespan"].cpu().numpy(), out["feasible"].cpu().numpy()
    fail = task.reward_spec.failing_signal
    rewards = [math.sqrt(m) if f else fail for m, f in zip(mk, fe)]
    assert row.mean_r == float(np.mean(rewards))
