"""The tcgen05 / TMA tensor-core paths against the fp64 DMMA kernels they
replace and against the CPU oracle.

The decoder weight gradient (``wgrad_tc.cu``: gw_dec, gb_dec and the
dev_table input-row terms of ``pkg/policy.py:378-395`` summed over samples as in
``pkg/trainer.py:138-154``) runs as int8 digit-plane MMAs with exact int32
accumulation in TMEM.  ``dp_debug_tensor_core(1)`` selects the DMMA kernel on
the same forward cache, so the two gradients are compared directly (norm-wise
relative 1e-12: the digit truncation is below 2^-45 per term), and the whole
gradient is checked against the oracle on weighted samples (1e-9, as the other
bench-size parity tests)."""

import numpy as np
import pytest
import torch

import paper_1706_04972_b200 as dp
from paper_1706_04972_b200 import _native as nat
from paper_1706_04972_b200 import policy as P
from test_bench_size_parity_gpu import GRAD_RTOL, _oracle_sum, _picks, _relnorm, _sampled, _setup, _weights

pytestmark = pytest.mark.gpu

AB_RTOL = 1e-12


@pytest.fixture(autouse=True)
def _tc_default():
    yield
    nat.check(nat.lib().dp_debug_tensor_core(0), "dp_debug_tensor_core")


def _grad(params, feats, K, seed, w, mode):
    """Sample K placements (fresh forward cache: the rows pass overwrites the
    gate activations with da in place) and run the trainer's split backward."""
    eng, pdev, pl, _ = _sampled(params, feats, K, seed)
    nat.check(nat.lib().dp_debug_tensor_core(mode), "dp_debug_tensor_core")
    adv = torch.as_tensor(w, device=eng.device)
    eng.backward_rows(pdev, K)
    g = eng.backward_grads(pdev, K, adv).cpu().numpy()
    nat.check(nat.lib().dp_debug_tensor_core(0), "dp_debug_tensor_core")
    return g


def _wdec_segments(params, g):
    """The gradient entries the decoder weight-gradient kernel produces."""
    lay = params.with_flat(g)
    return np.concatenate([lay.w_dec.ravel(), lay.b_dec.ravel(), lay.dev_table.ravel()])


@pytest.mark.parametrize("name,K,seed", [("C1", 8, 0), ("C1", 3, 1), ("C2", 64, 0), ("C3", 256, 0), ("C3tight", 40, 2)])
def test_dec_wgrad_tc_matches_dmma(name, K, seed):
    gg, topo, params, feats, pol = _setup(name, seed)
    w = np.random.default_rng(seed).normal(size=K) * 10.0 ** np.random.default_rng(seed + 1).uniform(-3, 3, K)
    g_tc = _grad(params, feats, K, seed + 5, w, 0)
    g_dm = _grad(params, feats, K, seed + 5, w, 1)
    assert _relnorm(_wdec_segments(params, g_tc), _wdec_segments(params, g_dm)) <= AB_RTOL
    assert _relnorm(g_tc, g_dm) <= AB_RTOL
    # the multi-segment epilogue (TMEM drained every 3 steps) gives the same sums
    g_seg = _grad(params, feats, K, seed + 5, w, 2)
    assert _relnorm(g_seg, g_dm) <= AB_RTOL


def test_dec_wgrad_tc_fused_backward_matches_dmma():
    """weighted_grad's fused pass (advantages folded into da: adv == NULL in the GEMM)."""
    gg, topo, params, feats, pol = _setup("C2", 3)
    w = np.random.default_rng(4).normal(size=48)
    out = []
    for mode in (0, 1):
        eng, pdev, pl, _ = _sampled(params, feats, 48, 9)
        nat.check(nat.lib().dp_debug_tensor_core(mode), "dp_debug_tensor_core")
        out.append(eng.backward(pdev, 48, torch.as_tensor(w, device=eng.device)).cpu().numpy())
    assert _relnorm(out[0], out[1]) <= AB_RTOL


def test_dec_wgrad_tc_zero_and_single_advantage():
    """All-zero advantages give an exactly zero gradient; one nonzero advantage
    reduces to that sample's grad log p (oracle)."""
    gg, topo, params, feats, pol = _setup("C1", 0)
    K = 16
    g0 = _grad(params, feats, K, 3, np.zeros(K), 0)
    assert not np.any(g0)
    w = np.zeros(K)
    w[5] = -2.5e-4
    g = _grad(params, feats, K, 3, w, 0)
    _, _, pl, _ = _sampled(params, feats, K, 3)
    assert _relnorm(g, _oracle_sum(pol, pl, w)) <= GRAD_RTOL


def test_dec_wgrad_tc_bench_size_vs_oracle():
    """C3 K=256 (the bench step) through the tensor-core path, against the oracle."""
    gg, topo, params, feats, pol = _setup("C3", 0)
    K = 256
    w = _weights(K, _picks(K, 2), seed=5)
    g = _grad(params, feats, K, 21, w, 0)
    _, _, pl, _ = _sampled(params, feats, K, 21)
    assert _relnorm(g, _oracle_sum(pol, pl, w)) <= GRAD_RTOL


@pytest.mark.parametrize("name,K,seed", [("C1", 8, 0), ("C2", 24, 1), ("C3", 256, 0), ("C3tight", 40, 2)])
def test_att_bwd_tc_matches_dmma_and_oracle(name, K, seed):
    """The attention backward on tcgen05 (att_tc.cu, debug mode 6): digit-plane
    dq = ds proj, A = alpha^T du, G = ds^T H against the DMMA kernel (1e-12)
    and the whole gradient against the oracle on weighted samples (1e-9)."""
    gg, topo, params, feats, pol = _setup(name, seed)
    w = np.random.default_rng(seed).normal(size=K) * 10.0 ** np.random.default_rng(seed + 1).uniform(-3, 3, K)
    g_tc = _grad(params, feats, K, seed + 5, w, 6)
    g_dm = _grad(params, feats, K, seed + 5, w, 1)
    assert _relnorm(g_tc, g_dm) <= AB_RTOL
    wo = _weights(K, _picks(K, 2), seed=5)
    g = _grad(params, feats, K, seed + 5, wo, 6)
    _, _, pl, _ = _sampled(params, feats, K, seed + 5)
    assert _relnorm(g, _oracle_sum(pol, pl, wo)) <= GRAD_RTOL
