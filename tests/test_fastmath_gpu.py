"""Accuracy of the branch-free fp64 transcendentals (csrc/fastmath.cuh) used by
the recurrent kernels, measured on the GPU against the CUDA libm in ulps.

The parity tests (bit-exact sampled placements and schedules, log-probs to
1e-12, gradients to 1e-9) absorb these few-ulp differences; this test pins
the bound so a faster but less accurate variant cannot slip in unnoticed."""

import ctypes

import pytest

pytestmark = pytest.mark.gpu


def test_fastmath_max_ulps():
    from paper_1706_04972_b200 import _native as nat

    out = (ctypes.c_uint64 * 5)()
    nat.check(nat.lib().dp_debug_fastmath_error(1 << 24, out), "dp_debug_fastmath_error")
    names = ["sigmoid", "tanh", "exp", "expm1", "div"]
    ulps = dict(zip(names, list(out)))
    print("fastmath max ulps:", ulps)
    assert ulps["div"] <= 1, ulps
    assert ulps["exp"] <= 2 and ulps["expm1"] <= 2, ulps
    assert ulps["sigmoid"] <= 4 and ulps["tanh"] <= 4, ulps
