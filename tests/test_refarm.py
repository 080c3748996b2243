"""The reference arm (oracle/refarm.py) runs genuine reference updates: its
pooled REINFORCE step reproduces the reference train()'s log (mean reward,
baseline) and its scorer the reference's makespans.  CPU only; skipped when the
reference install (oracle/make_ref.sh -> oracle/_ref) is absent."""

import os

import numpy as np
import pytest

from oracle import refarm

pytestmark = pytest.mark.skipif(not refarm.available(), reason="oracle/_ref not installed")
GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def test_pooled_step_matches_reference_train():
    path = os.path.join(GOLDEN, "cfg_C1.npz")
    ref, gg, topo = refarm.reference_instance(path)
    want = ref.trainer.train(gg, topo, ref.trainer.TrainerConfig(k=8, total_updates=3, seed=0))
    rs = refarm.RefStepper(path, 8, workers=3)
    try:
        got = []
        for _ in range(3):
            _, mean_r = rs.step()
            got.append((mean_r, rs.baseline.value))
    finally:
        rs.close()
    for row, (mean_r, base) in zip(want.log, got):
        assert mean_r == pytest.approx(row.mean_r, rel=1e-12)
        assert base == pytest.approx(row.baseline, rel=1e-12)
    np.testing.assert_allclose(rs.store.snapshot()[0], want.final_params, rtol=1e-9, atol=1e-12)


def test_scorer_matches_reference_simulate():
    path = os.path.join(GOLDEN, "cfg_C2.npz")
    r = refarm.scorer_rate(path, n=64, workers=3)
    ref, gg, topo = refarm.reference_instance(path)
    pl = np.random.default_rng(1).integers(0, topo.num_devices, (64, gg.num_groups))
    want = [ref.simulator.simulate(gg, topo, [int(x) for x in p]).makespan_seconds for p in pl]
    assert np.array_equal(r["makespans"], np.asarray(want))
