"""GPU parity of the policy kernels (csrc/policy_fwd.cu, policy_bwd.cu) through the C-ABI.

Bars (north_star): sampled indices / placements bit-exact; log-probs and
probabilities within 1e-12 relative (fp64 path; stated tolerance 1e-5);
gradients within 1e-9 norm-wise relative (stated tolerance 1e-5).
"""

import numpy as np
import pytest
import torch

from fixtures import cfg, npz
from oracle import policy as opol
import paper_1706_04972_b200 as dp
from paper_1706_04972_b200 import policy as P

pytestmark = pytest.mark.gpu

LP_RTOL = 1e-12
GRAD_RTOL = 1e-9


def _setup(name, seed=0):
    gg, topo, _, _ = cfg(name)
    tc = dp.TrainerConfig(seed=seed)
    params = dp.trainer.policy_template(gg, topo, tc)
    feats = P.GroupFeatures.from_grouped(gg, params.spec)
    return gg, topo, params, feats


def _rng_from(g):
    s = g["pcg_state"].astype(object)
    gen = np.random.Generator(np.random.PCG64())
    gen.bit_generator.state = {"bit_generator": "PCG64",
                               "state": {"state": (int(s[0]) << 64) | int(s[1]), "inc": (int(s[2]) << 64) | int(s[3])},
                               "has_uint32": 0, "uinteger": 0}
    return gen


def _relnorm(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300))


@pytest.mark.parametrize("name", ["C1", "C2", "C3"])
def test_forward_sample_matches_reference(name):
    gg, topo, params, feats = _setup(name)
    g = npz(f"policy_{name}.npz")
    assert np.array_equal(params.to_flat(), g["flat"])
    np.testing.assert_array_equal(P.embed_groups(params, feats), g["inputs"])
    rng = _rng_from(g)
    for k in range(len(g["placements"])):
        s = P.forward_sample(params, feats, rng)
        assert np.array_equal(s.placement, g["placements"][k]), f"sample {k} placement differs"
        assert s.log_prob == pytest.approx(g["log_probs"][k], rel=LP_RTOL)
    # the caller's generator advanced by exactly K*T draws
    ref_rng = _rng_from(g)
    ref_rng.bit_generator.advance(len(g["placements"]) * len(feats))
    assert rng.bit_generator.state == ref_rng.bit_generator.state


@pytest.mark.parametrize("name", ["C1", "C2", "C3"])
def test_teacher_forced_and_gradients_match_reference(name):
    gg, topo, params, feats = _setup(name)
    g = npz(f"policy_{name}.npz")
    pl0 = [int(x) for x in g["placements"][0]]
    np.testing.assert_allclose(P.step_distributions(params, feats, pl0), g["probs0"], rtol=1e-12, atol=1e-15)
    other = [int(x) for x in g["other"]]
    assert P.log_prob_of(params, feats, other) == pytest.approx(float(g["lp_other"]), rel=LP_RTOL)
    assert _relnorm(P.grad_log_prob(params, feats, pl0), g["grad0"]) < GRAD_RTOL
    assert _relnorm(P.grad_log_prob(params, feats, other), g["grad_other"]) < GRAD_RTOL


@pytest.mark.parametrize("name,K", [("C1", 64), ("C2", 32), ("C3", 48), ("C5", 3)])
def test_sample_batch_vs_oracle(name, K):
    """K samples in one launch == K sequential oracle forward_sample calls."""
    gg, topo, params, feats = _setup(name, seed=1)
    rng_a = np.random.default_rng(2024)
    rng_b = np.random.default_rng(2024)
    pl, lp = P.sample_batch(params, feats, rng_a, K)
    dims = opol.Dims(params.spec.table_rows, topo.num_devices)
    ofe = opol.features(gg, opol.vocab_of(gg))
    pol = opol.Policy(params.to_flat(), dims, ofe)
    for k in range(K):
        opl, olp, _ = pol.sample(rng_b)
        assert np.array_equal(pl[k], opl), f"sample {k}"
        assert lp[k] == pytest.approx(olp, rel=LP_RTOL)
    assert rng_a.bit_generator.state == rng_b.bit_generator.state


@pytest.mark.parametrize("name,K", [("C1", 16), ("C3", 8), ("C2", 5)])
def test_weighted_gradient_vs_oracle(name, K):
    gg, topo, params, feats = _setup(name, seed=3)
    pls = np.random.default_rng(5).integers(0, topo.num_devices, (K, gg.num_groups))
    w = np.random.default_rng(6).normal(size=K)
    got = P.weighted_grad(params, feats, [list(map(int, p)) for p in pls], w).cpu().numpy()
    dims = opol.Dims(params.spec.table_rows, topo.num_devices)
    pol = opol.Policy(params.to_flat(), dims, opol.features(gg, opol.vocab_of(gg)))
    ref = np.zeros(dims.n_params)
    for k in range(K):
        ref += w[k] * pol.grad([int(x) for x in pls[k]])
    assert _relnorm(got, ref) < GRAD_RTOL


@pytest.mark.parametrize("name,K", [("C3", 16), ("C2", 7)])
def test_split_backward_equals_fused(name, K):
    """rows (adv-independent, overlapped with scoring) + grads == fused single pass."""
    gg, topo, params, feats = _setup(name, seed=2)
    eng = P.engine_for(params, feats, K)
    pdev = torch.as_tensor(params.to_flat(), device=eng.device)
    eng.encode(pdev)
    eng.decode(pdev, K, pcg=(12345, 67891))
    adv = torch.as_tensor(np.random.default_rng(9).normal(size=K), device=eng.device)
    fused = eng.backward(pdev, K, adv).cpu().numpy()
    eng.decode(pdev, K, pcg=(12345, 67891))
    eng.backward_rows(pdev, K)
    split = eng.backward_grads(pdev, K, adv).cpu().numpy()
    assert _relnorm(split, fused) < 1e-12
    np.testing.assert_allclose(split, fused, rtol=1e-9, atol=1e-13)


def test_known_answers_zero_params_and_single_device():
    """zero params -> -T ln D ; D=1 -> log p = 0, zero gradient."""
    gg, topo, params, feats = _setup("C1")
    z = params.with_flat(np.zeros(params.flat_size))
    T = len(feats)
    assert P.log_prob_of(z, feats, [1] * T) == pytest.approx(-T * np.log(topo.num_devices), rel=1e-13)
    one = dp.DeviceTopology([dp.Device(0, "gpu", 1.0, 1 << 40)], [[0.0]])
    p1 = dp.trainer.policy_template(gg, one, dp.TrainerConfig())
    f1 = P.GroupFeatures.from_grouped(gg, p1.spec)
    s = P.forward_sample(p1, f1, np.random.default_rng(0))
    assert s.placement == [0] * T and s.log_prob == 0.0
    assert not np.any(P.grad_log_prob(p1, f1, s.placement))


def test_normalization_exhaustive_small():
    """Sum over all D^T placements of exp(log p) == 1, T=4, D=2."""
    ops = [dp.Operation(i, f"o{i}", "matmul" if i % 2 else "add", 1.0 + i, (4 + i,), 0) for i in range(4)]
    g = dp.ComputationGraph(ops, [dp.Edge(0, 1, 8), dp.Edge(1, 2, 8), dp.Edge(0, 3, 4)])
    gg = dp.singleton_groups(g)
    topo = dp.default_topology(1)
    params = dp.trainer.policy_template(gg, topo, dp.TrainerConfig(seed=4))
    feats = P.GroupFeatures.from_grouped(gg, params.spec)
    tot = 0.0
    for code in range(16):
        pl = [(code >> i) & 1 for i in range(4)]
        tot += np.exp(P.log_prob_of(params, feats, pl))
    assert abs(tot - 1.0) < 1e-12


def test_placement_validation_errors():
    gg, topo, params, feats = _setup("C1")
    with pytest.raises(ValueError, match="placement length"):
        P.log_prob_of(params, feats, [0, 1])
    with pytest.raises(ValueError, match="out of range"):
        P.grad_log_prob(params, feats, [topo.num_devices] * len(feats))


def test_checkpoint_roundtrip(tmp_path):
    gg, topo, params, feats = _setup("C1")
    P.save_checkpoint(params, tmp_path / "p.json")
    q = P.load_checkpoint(tmp_path / "p.json")
    assert np.array_equal(q.to_flat(), params.to_flat())
    torch.cuda.synchronize()


@pytest.mark.parametrize("name,K,picks", [("C1", 700, (0, 1, 349, 699)), ("C2", 600, (0, 599))])
def test_large_batch_non_speculative_decoder_vs_oracle(name, K, picks):
    """K > 4*148 selects the 8-samples-per-CTA decoder without the speculative
    cell (csrc/policy_fwd.cu plan_decoder); spot-check samples via PCG64 jumps."""
    gg, topo, params, feats = _setup(name, seed=4)
    T = len(feats)
    pl, lp = P.sample_batch(params, feats, np.random.default_rng(77), K)
    dims = opol.Dims(params.spec.table_rows, topo.num_devices)
    pol = opol.Policy(params.to_flat(), dims, opol.features(gg, opol.vocab_of(gg)))
    for k in picks:
        rng = np.random.default_rng(77)
        rng.bit_generator.advance(k * T)
        opl, olp, _ = pol.sample(rng)
        assert np.array_equal(pl[k], opl), f"sample {k}"
        assert lp[k] == pytest.approx(olp, rel=LP_RTOL)


@pytest.mark.parametrize("name,K", [("C3", 16), ("C2", 8), ("C1", 300)])
def test_speculative_cell_decoder_vs_oracle(name, K):
    """The opt-in speculative-cell decoder (dp_debug_decoder_variant(1)) samples
    the same placements as the oracle."""
    from paper_1706_04972_b200 import _native as nat

    gg, topo, params, feats = _setup(name, seed=5)
    nat.check(nat.lib().dp_debug_decoder_variant(1), "variant")
    try:
        pl, lp = P.sample_batch(params, feats, np.random.default_rng(11), K)
    finally:
        nat.check(nat.lib().dp_debug_decoder_variant(0), "variant")
    dims = opol.Dims(params.spec.table_rows, topo.num_devices)
    pol = opol.Policy(params.to_flat(), dims, opol.features(gg, opol.vocab_of(gg)))
    rng = np.random.default_rng(11)
    for k in range(min(K, 16)):
        opl, olp, _ = pol.sample(rng)
        assert np.array_equal(pl[k], opl), f"sample {k}"
        assert lp[k] == pytest.approx(olp, rel=LP_RTOL)


@pytest.mark.parametrize("name,K,n_check", [("C3", 16, 16), ("C1", 8, 8), ("C5", 4, 2)])
def test_cluster_encoder_vs_oracle(name, K, n_check):
    """The opt-in 4-CTA cluster encoder recurrence (dp_debug_encoder_variant(1):
    DSMEM h exchange through st.async + mbarrier transaction counts) samples the
    oracle's placements and matches its log-probs and gradient."""
    from paper_1706_04972_b200 import _native as nat

    gg, topo, params, feats = _setup(name, seed=23)  # a seed no other test encodes (engine cache)
    nat.check(nat.lib().dp_debug_encoder_variant(1), "variant")
    try:
        pl, lp = P.sample_batch(params, feats, np.random.default_rng(17), K)
        got = P.grad_log_prob(params, feats, [int(x) for x in pl[0]])
    finally:
        nat.check(nat.lib().dp_debug_encoder_variant(0), "variant")
    dims = opol.Dims(params.spec.table_rows, topo.num_devices)
    pol = opol.Policy(params.to_flat(), dims, opol.features(gg, opol.vocab_of(gg)))
    rng = np.random.default_rng(17)
    for k in range(n_check):
        opl, olp, _ = pol.sample(rng)
        assert np.array_equal(pl[k], opl), f"sample {k}"
        assert lp[k] == pytest.approx(olp, rel=LP_RTOL)
    assert _relnorm(got, pol.grad([int(x) for x in pl[0]])) < 1e-8


@pytest.mark.parametrize("scale", [1.0, 400.0])
def test_attention_softmax_shift_paths_vs_oracle(scale):
    """Large attention weights (8 max||proj_t|| > 600) take the max-shifted
    softmax; small ones the shift-free path (csrc/policy_fwd.cu kNoShiftBound).
    Both sample the oracle's placements and match its log-probs and gradient."""
    gg, topo, params, feats = _setup("C1", seed=6)
    params.w_att = params.w_att * scale
    pl, lp = P.sample_batch(params, feats, np.random.default_rng(3), 6)
    dims = opol.Dims(params.spec.table_rows, topo.num_devices)
    pol = opol.Policy(params.to_flat(), dims, opol.features(gg, opol.vocab_of(gg)))
    rng = np.random.default_rng(3)
    for k in range(6):
        opl, olp, _ = pol.sample(rng)
        assert np.array_equal(pl[k], opl), f"sample {k}"
        assert lp[k] == pytest.approx(olp, rel=1e-10)
    got = P.grad_log_prob(params, feats, [int(x) for x in pl[0]])
    assert _relnorm(got, pol.grad([int(x) for x in pl[0]])) < 1e-8


@pytest.mark.parametrize("name,K,picks", [("C3", 256, (0, 1, 127, 255)), ("C5", 4096, (0, 2049, 4095))])
def test_bench_size_decoder_vs_oracle(name, K, picks):
    """The decoder instantiations bench.py times (C3 K=256: 2 samples per CTA,
    FAST path; C5 K=4096: 8 samples per CTA, DM path) at their full sizes:
    oracle spot checks via PCG64 jumps, and the size-independent property that
    the teacher-forced pass over the whole sampled batch reproduces every
    sampled log-probability."""
    gg, topo, params, feats = _setup(name, seed=6)
    T = len(feats)
    pl, lp = P.sample_batch(params, feats, np.random.default_rng(91), K)
    assert pl.shape == (K, T) and np.isfinite(lp).all() and (lp <= 0).all()
    assert pl.min() >= 0 and pl.max() < topo.num_devices
    dims = opol.Dims(params.spec.table_rows, topo.num_devices)
    pol = opol.Policy(params.to_flat(), dims, opol.features(gg, opol.vocab_of(gg)))
    for k in picks:
        rng = np.random.default_rng(91)
        rng.bit_generator.advance(k * T)
        opl, olp, _ = pol.sample(rng)
        assert np.array_equal(pl[k], opl), f"sample {k}"
        assert lp[k] == pytest.approx(olp, rel=LP_RTOL)
    with P._locked_tf(params, feats, [list(r) for r in pl]) as (_, _, tlp, _):
        np.testing.assert_allclose(tlp.cpu().numpy(), lp, rtol=LP_RTOL, atol=0)


def test_dropin_calls_from_threads_share_one_engine():
    """Controller threads of the reference (pkg/trainer.py:365-378) call the
    drop-in functions concurrently on one GroupFeatures object: the per-engine
    lock keeps each encode -> decode -> backward sequence intact."""
    import threading

    gg, topo, params, feats = _setup("C1", seed=2)
    dims = opol.Dims(params.spec.table_rows, topo.num_devices)
    pol = opol.Policy(params.to_flat(), dims, opol.features(gg, opol.vocab_of(gg)))
    errors = []

    def worker(seed):
        try:
            rng, orng = np.random.default_rng(seed), np.random.default_rng(seed)
            for _ in range(6):
                s = P.forward_sample(params, feats, rng)
                opl, olp, _ = pol.sample(orng)
                assert s.placement == opl
                g = P.grad_log_prob(params, feats, s.placement, cache=s.cache)
                assert _relnorm(g, pol.grad(opl)) < GRAD_RTOL
                assert P.log_prob_of(params, feats, s.placement) == pytest.approx(olp, rel=LP_RTOL)
        except Exception as ex:  # surfaced below
            errors.append(repr(ex))

    ths = [threading.Thread(target=worker, args=(100 + i,)) for i in range(4)]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    assert not errors, errors


def test_dropin_encoder_cache_follows_parameter_changes():
    """forward_sample / grad_log_prob reuse the engine's encoder while the
    caller's parameters are unchanged (content compare); a new snapshot, an
    in-place edit of the same object, or a batched call that re-encodes
    in between must all be honoured (oracle at every step)."""
    gg, topo, params, feats = _setup("C2", seed=4)
    dims = opol.Dims(params.spec.table_rows, topo.num_devices)
    vocab = opol.vocab_of(gg)

    def oracle_for(p):
        return opol.Policy(p.to_flat(), dims, opol.features(gg, vocab))

    p2 = params.with_flat(params.to_flat() * 1.7)
    for cur in (params, p2, params):
        pol = oracle_for(cur)
        rng, orng = np.random.default_rng(9), np.random.default_rng(9)
        for _ in range(3):
            s = P.forward_sample(cur, feats, rng)
            opl, olp, _ = pol.sample(orng)
            assert s.placement == opl and s.log_prob == pytest.approx(olp, rel=LP_RTOL)
        assert _relnorm(P.grad_log_prob(cur, feats, s.placement, cache=s.cache), pol.grad(opl)) < GRAD_RTOL
        # a batched call on the same engine re-encodes other parameters in between
        P.sample_batch(p2 if cur is params else params, feats, np.random.default_rng(1), 3)
        assert P.log_prob_of(cur, feats, s.placement) == pytest.approx(olp, rel=LP_RTOL)
    # in-place edit of the same PolicyParams object
    params.w_att *= 0.5
    pol = oracle_for(params)
    rng, orng = np.random.default_rng(5), np.random.default_rng(5)
    s = P.forward_sample(params, feats, rng)
    opl, olp, _ = pol.sample(orng)
    assert s.placement == opl and s.log_prob == pytest.approx(olp, rel=LP_RTOL)


def _decoder_plan(eng, K):
    import ctypes

    from paper_1706_04972_b200 import _native as nat

    out = (ctypes.c_int32 * 6)()
    nat.check(nat.lib().dp_debug_decoder_plan(eng.handle, K, out), "plan")
    return dict(zip(["M", "MT", "tcg", "smem", "spec", "enc_in_smem"], list(out)))


@pytest.mark.parametrize("name,K", [("C3", 256), ("C1", 100), ("C1", 290)])
def test_tensor_core_gates_decoder(name, K):
    """The opt-in FAST decoder with its gate mat-vec h W_h on tcgen05 (int8
    digit planes of W_h resident in TMEM, csrc/policy_fwd.cu TCG,
    dp_debug_decoder_variant(4)) against the default fp64-pipe mat-vec:
    identical placements, log-probs within 1e-12, per-step probabilities within
    1e-13, weighted gradients within 1e-10; and the oracle's placements /
    log-probs for the first samples."""
    from paper_1706_04972_b200 import _native as nat

    gg, topo, params, feats = _setup(name, seed=4)
    eng = P.engine_for(params, feats, K)
    assert _decoder_plan(eng, K)["tcg"] == 0
    pl3, lp3 = P.sample_batch(params, feats, np.random.default_rng(21), K)
    w = np.linspace(-1.0, 1.0, 8)
    g3 = P.weighted_grad(params, feats, [list(map(int, p)) for p in pl3[:8]], w).cpu().numpy()
    pr3 = P.step_distributions(params, feats, list(map(int, pl3[0])))
    nat.check(nat.lib().dp_debug_decoder_variant(4), "variant")
    try:
        plan = _decoder_plan(eng, K)
        assert plan["tcg"] == 1 and plan["MT"] <= 2, plan
        pl, lp = P.sample_batch(params, feats, np.random.default_rng(21), K)
        g = P.weighted_grad(params, feats, [list(map(int, p)) for p in pl[:8]], w).cpu().numpy()
        pr = P.step_distributions(params, feats, list(map(int, pl[0])))
    finally:
        nat.check(nat.lib().dp_debug_decoder_variant(0), "variant")
    assert np.array_equal(pl, pl3)
    np.testing.assert_allclose(lp, lp3, rtol=LP_RTOL, atol=0)
    assert _relnorm(g, g3) <= 1e-10
    assert np.max(np.abs(pr - pr3)) <= 1e-13
    dims = opol.Dims(params.spec.table_rows, topo.num_devices)
    pol = opol.Policy(params.to_flat(), dims, opol.features(gg, opol.vocab_of(gg)))
    rng = np.random.default_rng(21)
    for k in range(4):
        opl, olp, _ = pol.sample(rng)
        assert np.array_equal(pl[k], opl), f"sample {k}"
        assert lp[k] == pytest.approx(olp, rel=LP_RTOL)
