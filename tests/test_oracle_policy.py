"""Pin the CPU policy / RNG / trainer oracle to reference-generated goldens."""

import numpy as np
import pytest

from fixtures import cfg, npz, train_golden
from oracle import pcg64
from oracle import policy as opol
from oracle import trainer as otr


def _setup(name):
    gg, topo, _, _ = cfg(name)
    dims = opol.Dims(len(opol.vocab_of(gg)) + 1, topo.num_devices)
    feats = opol.features(gg, opol.vocab_of(gg))
    return gg, topo, dims, feats


def _rng(g):
    s = g["pcg_state"].astype(object)
    state = (int(s[0]) << 64) | int(s[1])
    inc = (int(s[2]) << 64) | int(s[3])
    gen = np.random.Generator(np.random.PCG64())
    gen.bit_generator.state = {"bit_generator": "PCG64", "state": {"state": state, "inc": inc},
                               "has_uint32": 0, "uinteger": 0}
    return gen, state, inc


@pytest.mark.parametrize("name", ["C1", "C2", "C3"])
def test_policy_oracle_matches_reference(name):
    gg, topo, dims, feats = _setup(name)
    g = npz(f"policy_{name}.npz")
    assert list(g["vocab"]) == opol.vocab_of(gg)
    flat = opol.init_flat(dims, 0)
    assert np.array_equal(flat, g["flat"])
    pol = opol.Policy(flat, dims, feats)
    assert np.array_equal(pol.inputs(), g["inputs"])
    gen, _, _ = _rng(g)
    for k in range(len(g["placements"])):
        pl, lp, tape = pol.sample(gen)
        assert np.array_equal(pl, g["placements"][k])
        assert lp == g["log_probs"][k]
        if k == 0:
            assert np.array_equal(pol.step_probs(pl), g["probs0"])
            np.testing.assert_allclose(pol.grad(pl, tape), g["grad0"], rtol=1e-12, atol=1e-15)
    other = [int(x) for x in g["other"]]
    assert pol.log_prob(other) == g["lp_other"]
    np.testing.assert_allclose(pol.grad(other), g["grad_other"], rtol=1e-12, atol=1e-15)


def test_pcg64_restatement_matches_numpy():
    gen = np.random.default_rng(np.random.SeedSequence(0).spawn(1)[0].spawn(2)[0])
    state, inc = pcg64.state_of(gen)
    draws = gen.random(3000)
    for n in list(range(50)) + [999, 2999]:
        assert pcg64.random_at(state, inc, n) == draws[n]
    gen2 = np.random.default_rng(5)
    s2, i2 = pcg64.state_of(gen2)
    gen2.bit_generator.advance(1_000_003)
    assert pcg64.state_of(gen2)[0] == pcg64.jump(s2, i2, 1_000_003)


def test_policy_known_answers():
    """zero params -> -T ln D; D=1 -> 0 and zero gradient."""
    gg, topo, dims, feats = _setup("C1")
    pol = opol.Policy(np.zeros(dims.n_params), dims, feats)
    T = gg.num_groups
    assert pol.log_prob([0] * T) == pytest.approx(-T * np.log(topo.num_devices), rel=1e-13)


@pytest.mark.parametrize("name", ["C1", "C3tight", "C2"])
def test_trainer_oracle_matches_reference(name):
    gg, topo, _, _ = cfg(name)
    g = train_golden(name)
    out = otr.run(gg, topo, g["cfg"], record=True)
    assert otr.csv_of(out["rows"]) == g["csv"]
    assert np.array_equal(np.array(out["placements"], np.uint8), g["placements"])
    assert np.array_equal(np.array(out["measure"]), g["measure"])
    for mine, ref in zip(out["grads"], g["grads"]):
        if mine is None:
            assert np.isnan(ref).all()
        else:
            np.testing.assert_allclose(mine, ref, rtol=1e-10, atol=1e-14)
    np.testing.assert_allclose(out["final"], g["final_params"], rtol=1e-12, atol=1e-15)
    assert out["versions"] == int(g["store_versions"])
    if out["best_placement"] is not None:
        assert np.array_equal(out["best_placement"], g["best_placement"])


@pytest.mark.parametrize("name,graph", [("C1noise", "C1"), ("C3noise", "C3tight")])
def test_trainer_oracle_with_measurement_noise_matches_reference(name, graph):
    """f2: lognormal measurement noise (reference train() with noise_sigma > 0)."""
    gg, topo, _, _ = cfg(graph)
    g = train_golden(name)
    out = otr.run(gg, topo, g["cfg"], record=True)
    assert otr.csv_of(out["rows"]) == g["csv"]
    assert np.array_equal(np.array(out["placements"], np.uint8), g["placements"])
    np.testing.assert_allclose(out["final"], g["final_params"], rtol=1e-12, atol=1e-15)
    assert out["versions"] == int(g["store_versions"])


def test_trainer_oracle_round_schedule_single_controller_is_run():
    """run_multi (the f1 round schedule) with one controller == the pinned run()."""
    gg, topo, _, _ = cfg("C1")
    g = train_golden("C1")
    out = otr.run_multi(gg, topo, g["cfg"])
    assert otr.csv_of(out["rows"]) == g["csv"]
    np.testing.assert_allclose(out["final"], g["final_params"], rtol=1e-12, atol=1e-15)
