"""Gradient and sampling parity at the batch sizes bench.py runs.

The kernels the benchmark configurations select differ from the small-K ones:

* decoder LSTM backward ``lstm_bwd_kernel<M>`` with M = ceil(K/148) samples per
  CTA (policy_bwd.cu ``run_b2``): M=2 at C3 K=256, M=3..4 (the <4>
  instantiation) at C4 K=512 and above;
* attention backward: GM mode with stored numerators in the split (trainer)
  backward, stored-numerator fused mode in ``weighted_grad``, and the
  score-recompute ``att_bwd_kernel<false>`` when the numerators do not fit
  (C5 K=4096) — forced at small K with ``dp_debug_policy_drop_stores``;
* the non-speculative 4-samples-per-CTA decoder at K=512 (C4's tasks).

Each check compares against the CPU oracle (``oracle/policy.py``, pinned to the
reference in tests/test_oracle_policy.py): sum_k w_k grad log p_k with nonzero
weights on a spread of samples (every position inside a CTA, CTA boundaries,
first/last sample) and zero on the rest, so the oracle stays cheap while every
kernel runs at full size.  Reference: ``pkg/policy.py:351-409`` (grad_log_prob),
``pkg/trainer.py:138-154`` (the weighted sum).  Tolerance: norm-wise relative
1e-9 (stated bar 1e-5).
"""

import numpy as np
import pytest
import torch

from fixtures import cfg
from oracle import policy as opol
import paper_1706_04972_b200 as dp
from paper_1706_04972_b200 import _native as nat
from paper_1706_04972_b200 import policy as P

pytestmark = pytest.mark.gpu

GRAD_RTOL = 1e-9
LP_RTOL = 1e-12


def _setup(name, seed):
    gg, topo, _, _ = cfg(name)
    params = dp.trainer.policy_template(gg, topo, dp.TrainerConfig(seed=seed))
    feats = P.GroupFeatures.from_grouped(gg, params.spec)
    dims = opol.Dims(params.spec.table_rows, topo.num_devices)
    pol = opol.Policy(params.to_flat(), dims, opol.features(gg, opol.vocab_of(gg)))
    return gg, topo, params, feats, pol


def _picks(K, M):
    """Samples to weight: every slot of the first/last CTA (M samples each), the
    slots around the middle CTA boundary, and a few strided ones."""
    s = set(range(min(M, K))) | set(range(max(0, K - M), K))
    mid = (K // (2 * M)) * M
    s |= {x for x in range(mid - 2, mid + M + 2) if 0 <= x < K}
    s |= set(range(0, K, max(1, K // 8)))
    return sorted(s)


def _weights(K, picks, seed=11):
    w = np.zeros(K)
    w[picks] = np.random.default_rng(seed).normal(size=len(picks))
    return w


def _oracle_sum(pol, placements, w):
    ref = np.zeros(pol.dims.n_params)
    for k in np.nonzero(w)[0]:
        ref += w[k] * pol.grad([int(x) for x in placements[k]])
    return ref


def _relnorm(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300))


def _split_grad(eng, pdev, K, w):
    """The trainer's backward: rows pass (advantage-independent) + grads pass."""
    adv = torch.as_tensor(w, device=eng.device)
    eng.backward_rows(pdev, K)
    return eng.backward_grads(pdev, K, adv).cpu().numpy()


def _sampled(params, feats, K, seed):
    """Sample K placements on the device (leaves the engine's forward cache in
    place for the split backward, exactly as the trainer does)."""
    eng = P.engine_for(params, feats, K)
    pdev = torch.as_tensor(params.to_flat(), device=eng.device)
    eng.encode(pdev)
    choice, lp = eng.decode(pdev, K, pcg=P.generator_state(np.random.default_rng(seed)))
    return eng, pdev, eng.by_gid(choice).cpu().numpy(), lp.cpu().numpy()


# lstm_bwd_kernel<2> (K=160: M=2), <4> with M=3 (K=320) and M=4 (K=600)
@pytest.mark.parametrize("name,K", [("C1", 160), ("C1", 320), ("C2", 600)])
def test_weighted_grad_large_k_vs_oracle(name, K):
    gg, topo, params, feats, pol = _setup(name, seed=3)
    M = min(4, -(-K // 148))
    pls = np.random.default_rng(5).integers(0, topo.num_devices, (K, gg.num_groups))
    w = _weights(K, _picks(K, M))
    got = P.weighted_grad(params, feats, [list(map(int, p)) for p in pls], w).cpu().numpy()
    assert _relnorm(got, _oracle_sum(pol, pls, w)) < GRAD_RTOL


@pytest.mark.parametrize("name,K", [("C3", 256), ("C1", 320), ("C2", 512)])
def test_trainer_split_backward_bench_size_vs_oracle(name, K):
    """The trainer's exact sequence at bench sizes: sample K on the device, rows
    pass (GM attention backward from the stored numerators, lstm_bwd<M>), then
    the advantage-weighted grads pass."""
    gg, topo, params, feats, pol = _setup(name, seed=4)
    eng, pdev, pls, lp = _sampled(params, feats, K, seed=21)
    M = min(4, -(-K // 148))
    w = _weights(K, _picks(K, M), seed=12)
    got = _split_grad(eng, pdev, K, w)
    assert _relnorm(got, _oracle_sum(pol, pls, w)) < GRAD_RTOL
    # the same batch through the fused single pass agrees to rounding
    fused = P.weighted_grad(params, feats, [list(map(int, p)) for p in pls], w).cpu().numpy()
    assert _relnorm(fused, got) < 1e-12


@pytest.mark.parametrize("mask", [1, 2, 3])
@pytest.mark.parametrize("name,K", [("C3", 16), ("C2", 7), ("C1", 160)])
def test_dropped_stores_backward_vs_oracle(name, K, mask):
    """Engines without stored attention numerators (mask 1: att_bwd<false>, score
    recompute) and/or without per-tile partials (mask 2: the rows pass is
    skipped and the grads call runs the fused backward) — the paths C5 K=4096
    takes — against the oracle, through both the split and fused entry points."""
    gg, topo, params, feats, pol = _setup(name, seed=7)
    eng = P.DevicePolicy(feats, params.spec, topo.num_devices, k_max=K)
    nat.check(nat.lib().dp_debug_policy_drop_stores(eng.handle, mask), "drop_stores")
    pdev = torch.as_tensor(params.to_flat(), device=eng.device)
    eng.encode(pdev)
    choice, _ = eng.decode(pdev, K, pcg=P.generator_state(np.random.default_rng(31)))
    pls = eng.by_gid(choice).cpu().numpy()
    w = _weights(K, _picks(K, min(4, -(-K // 148))), seed=13)
    ref = _oracle_sum(pol, pls, w)
    assert _relnorm(_split_grad(eng, pdev, K, w), ref) < GRAD_RTOL
    adv = torch.as_tensor(w, device=eng.device)
    eng.decode(pdev, K, forced=P._forced_by_rank(eng, feats, pls))
    assert _relnorm(eng.backward(pdev, K, adv).cpu().numpy(), ref) < GRAD_RTOL


def test_c5_full_batch_backward_vs_oracle():
    """C5 at its bench size (T=2000, K=4096): the decoder's DM path, no stored
    numerators and no tile partials (too large), so the trainer's backward is
    the fused score-recompute pass.  Weighted on three samples."""
    gg, topo, params, feats, pol = _setup("C5", seed=6)
    K = 4096
    eng, pdev, pls, lp = _sampled(params, feats, K, seed=41)
    w = np.zeros(K)
    w[[0, 2049, 4095]] = [0.7, -1.3, 0.4]
    got = _split_grad(eng, pdev, K, w)
    assert _relnorm(got, _oracle_sum(pol, pls, w)) < GRAD_RTOL


@pytest.mark.parametrize("name,K,picks", [("C1", 512, (0, 3, 4, 255, 256, 511)),
                                          ("C2", 512, (0, 1, 2, 3, 300, 511)),
                                          ("C3", 300, (0, 3, 4, 150, 299))])
def test_four_per_cta_decoder_vs_oracle(name, K, picks):
    """K in (296, 592] selects M=4 samples per CTA without the speculative cell
    (C4's tasks at K=512); spot checks through PCG64 jumps to each sample's
    draw index k*T, plus the teacher-forced log-probs of the whole batch."""
    gg, topo, params, feats, pol = _setup(name, seed=8)
    T = len(feats)
    pl, lp = P.sample_batch(params, feats, np.random.default_rng(55), K)
    for k in picks:
        rng = np.random.default_rng(55)
        rng.bit_generator.advance(k * T)
        opl, olp, _ = pol.sample(rng)
        assert np.array_equal(pl[k], opl), f"sample {k}"
        assert lp[k] == pytest.approx(olp, rel=LP_RTOL)
    with P._locked_tf(params, feats, [list(r) for r in pl]) as (_, _, tlp, _):
        np.testing.assert_allclose(tlp.cpu().numpy(), lp, rtol=LP_RTOL, atol=0)


def _oracle_sample_with_margin(pol, rng):
    """The reference sampling rule (pkg/policy.py:320-323) recording each draw's
    distance to the cdf boundaries that can change the index (j < D-1)."""
    D = pol.dims.n_dev
    margin = [np.inf]
    pdiff_probs = []

    def pick(_t, probs):
        r = rng.random()
        cdf = np.cumsum(probs)
        if D > 1:
            margin[0] = min(margin[0], float(np.min(np.abs(r - cdf[:D - 1]))))
        pdiff_probs.append(probs)
        return min(int(np.searchsorted(cdf, r, side="right")), D - 1)

    pl, lp, _ = pol.run(pick)
    return pl, lp, margin[0], np.stack(pdiff_probs)


@pytest.mark.parametrize("name,K,picks", [("C1", 64, (0, 17, 63)), ("C2", 64, (0, 40)),
                                          ("C3", 256, (0, 1, 128, 255)), ("C5", 512, (0, 511))])
def test_sampling_margin_certificate(name, K, picks):
    """dp_policy_decode's margin output equals the oracle's per-sample
    min |r - cdf_j| (to 1e-12), every spot-checked draw is far from a boundary
    compared with the device-vs-oracle distribution difference, and at these
    seeds no sample is uncertified (margin < SAMPLING_MARGIN_TOL)."""
    gg, topo, params, feats, pol = _setup(name, seed=9)
    T = len(feats)
    pl, lp, margin = P.sample_batch(params, feats, np.random.default_rng(123), K, return_margin=True)
    assert margin.shape == (K,) and np.all(margin >= 0)
    worst_pdiff = 0.0
    for k in picks:
        rng = np.random.default_rng(123)
        rng.bit_generator.advance(k * T)
        opl, olp, omg, oprobs = _oracle_sample_with_margin(pol, rng)
        assert np.array_equal(pl[k], opl), f"sample {k}"
        assert abs(margin[k] - omg) <= 1e-12, (k, margin[k], omg)
        dprobs = P.step_distributions(params, feats, [int(x) for x in pl[k]])
        worst_pdiff = max(worst_pdiff, float(np.max(np.abs(dprobs - oprobs))))
    assert worst_pdiff < 1e-12
    assert margin.min() > P.SAMPLING_MARGIN_TOL > 1e3 * worst_pdiff


def test_single_device_margin_is_infinite():
    gg, topo, _, _ = cfg("C1")
    one = dp.DeviceTopology([dp.Device(0, "gpu", 1.0, 1 << 40)], [[0.0]])
    p1 = dp.trainer.policy_template(gg, one, dp.TrainerConfig())
    f1 = P.GroupFeatures.from_grouped(gg, p1.spec)
    _, _, m = P.sample_batch(p1, f1, np.random.default_rng(0), 3, return_margin=True)
    assert np.all(np.isinf(m))


def test_trainer_reports_sampling_certificate():
    gg, topo, _, _ = cfg("C3")
    res = dp.train(gg, topo, dp.TrainerConfig(k=64, total_updates=3, seed=2))
    cert = res.sampling
    assert cert["uncertified_samples"] == 0 and cert["min_margin"] > cert["tol"]


def test_margin_accumulate_kernel():
    """dp_margin_accumulate (the trainer's per-update sampling certificate):
    running minimum of the per-sample margins and the count below tol, over
    several launches and a K that spans several warps."""
    import ctypes

    from paper_1706_04972_b200 import _native as nat

    rng = np.random.default_rng(5)
    mm = torch.full((1,), np.inf, dtype=torch.float64, device="cuda")
    nb = torch.zeros(1, dtype=torch.int64, device="cuda")
    want_min, want_n = np.inf, 0
    for K in (1, 37, 300, 4096):
        m = rng.uniform(0.0, 1e-8, K) * (rng.random(K) < 0.5) + rng.uniform(1e-6, 1.0, K) * 0.5
        m[rng.integers(0, K)] = np.inf
        md = torch.as_tensor(m, device="cuda")
        nat.check(nat.lib().dp_margin_accumulate(K, nat.ptr(md), ctypes.c_double(1e-7), nat.ptr(mm), nat.ptr(nb),
                                                 nat.stream_ptr()), "dp_margin_accumulate")
        want_min = min(want_min, float(np.min(m)))
        want_n += int(np.sum(m < 1e-7))
    torch.cuda.synchronize()
    assert float(mm.item()) == want_min and int(nb.item()) == want_n


@pytest.mark.parametrize("ngpu,K,picks", [(5, 7, (0, 6)),            # D=6, 1 sample per CTA
                                          (7, 200, (0, 1, 199)),     # D=8, 2 per CTA
                                          (7, 297, (0, 3, 295, 296)),  # D=8, 4 per CTA, last CTA holds 1
                                          (3, 297, (0, 296))])       # D=4, 4 per CTA, last CTA holds 1
def test_fast_decoder_device_and_sample_bounds_vs_oracle(ngpu, K, picks):
    """The FAST decoder instantiations at their bounds — up to 8 devices (4 logit
    lanes per device, 24-double step records) and 4 samples per CTA including a
    partial last CTA — against the oracle: placements bit-exact, log-probs and a
    weighted gradient over the picked samples."""
    from paper_1706_04972_b200 import _native as nat  # noqa: F401

    gg, _, _, _ = cfg("C1")
    topo = dp.simulator.default_topology(num_gpus=ngpu)
    params = dp.trainer.policy_template(gg, topo, dp.TrainerConfig(seed=13))
    feats = P.GroupFeatures.from_grouped(gg, params.spec)
    dims = opol.Dims(params.spec.table_rows, topo.num_devices)
    pol = opol.Policy(params.to_flat(), dims, opol.features(gg, opol.vocab_of(gg)))
    T = len(feats)
    pl, lp = P.sample_batch(params, feats, np.random.default_rng(31), K)
    assert pl.max() < topo.num_devices
    for k in picks:
        rng = np.random.default_rng(31)
        rng.bit_generator.advance(k * T)
        opl, olp, _ = pol.sample(rng)
        assert np.array_equal(pl[k], opl), f"sample {k}"
        assert lp[k] == pytest.approx(olp, rel=LP_RTOL)
    w = np.zeros(K)
    w[list(picks)] = np.linspace(0.5, -0.75, len(picks))
    got = P.weighted_grad(params, feats, [list(map(int, p)) for p in pl], w).cpu().numpy()
    assert _relnorm(got, _oracle_sum(pol, pl, w)) < GRAD_RTOL
