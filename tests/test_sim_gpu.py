"""GPU parity of the K-sim kernel (csrc/sim.cu) through the C-ABI.

Bar: bit-exact makespan / busy / transfer / peak / feasible / dispatch order
against the reference (goldens) and the CPU oracle.
"""

import numpy as np
import pytest
import torch

from fixtures import cfg, npz, random_cases
from oracle.sim import OracleGraph
import paper_1706_04972_b200.simulator as S

pytestmark = pytest.mark.gpu
CONFIGS = ["C1", "C2", "C3", "C3tight", "C5"]


@pytest.fixture(params=["warp", "thread"], autouse=True)
def sim_variant(request):
    """Every test runs on both simulator kernels: one warp per placement and
    one thread per placement (dp_debug_sim_variant)."""
    from paper_1706_04972_b200 import _native as nat

    nat.check(nat.lib().dp_debug_sim_variant(1 if request.param == "warp" else 2), "variant")
    yield request.param
    nat.check(nat.lib().dp_debug_sim_variant(0), "variant")


def _host(out):
    return {k: v.cpu().numpy() for k, v in out.items()}


@pytest.mark.parametrize("name", CONFIGS)
def test_sim_kernel_matches_reference_goldens(name):
    gg, topo, _, _ = cfg(name)
    g = npz(f"sim_{name}.npz")
    out = _host(S.simulate_batch(gg, topo, g["placements"], order=True))
    assert out["err"][0] == 0
    for k in ("makespan", "busy", "transfer", "peak", "feasible", "order"):
        assert np.array_equal(out[k], g[k]), k


def test_sim_kernel_random_suite_incl_zero_costs():
    for gg, topo, pl, exp in random_cases():
        out = _host(S.simulate_batch(gg, topo, [pl], order=True))
        assert out["makespan"][0] == exp["makespan"]
        assert np.array_equal(out["busy"][0], exp["busy"])
        assert np.array_equal(out["transfer"][0], exp["transfer"])
        assert np.array_equal(out["peak"][0], exp["peak"])
        assert bool(out["feasible"][0]) == exp["feasible"]
        assert np.array_equal(out["order"][0], exp["order"])


@pytest.mark.parametrize("name,K", [("C1", 4096), ("C2", 2048), ("C3", 4096), ("C3tight", 1024), ("C5", 512)])
def test_sim_kernel_large_batch_vs_oracle(name, K):
    gg, topo, _, _ = cfg(name)
    pl = np.random.default_rng(11).integers(0, topo.num_devices, (K, gg.num_groups))
    out = _host(S.simulate_batch(gg, topo, pl, order=True))
    ref = OracleGraph(gg, topo).simulate(pl, order=True, threads=8)
    for k in ("makespan", "busy", "transfer", "peak", "feasible", "order"):
        assert np.array_equal(out[k], ref[k]), k


def test_by_rank_layout_equivalent():
    gg, topo, _, _ = cfg("C2")
    pl = np.random.default_rng(3).integers(0, topo.num_devices, (64, gg.num_groups)).astype(np.uint8)
    by_rank = pl[:, np.asarray(gg.topo)]
    a = _host(S.simulate_batch(gg, topo, pl))
    b = _host(S.simulate_batch(gg, topo, by_rank, by_rank=True))
    for k in ("makespan", "busy", "transfer", "peak", "feasible"):
        assert np.array_equal(a[k], b[k])


def test_invalid_device_flags_error():
    gg, topo, _, _ = cfg("C1")
    pl = np.zeros((3, gg.num_groups), np.uint8)
    pl[1, 5] = topo.num_devices
    out = _host(S.simulate_batch(gg, topo, pl))
    assert out["err"][0] == 1 and np.isnan(out["makespan"][1]) and not np.isnan(out["makespan"][0])
    with pytest.raises(ValueError, match="out of range"):
        S.simulate(gg, topo, [0] * (gg.num_groups - 1) + [topo.num_devices])
    with pytest.raises(ValueError, match="placement length"):
        S.simulate(gg, topo, [0] * 3)


def test_dropin_simulate_measure_check_memory():
    gg, topo, _, _ = cfg("C3tight")
    g = npz("sim_C3tight.npz")
    for k in range(4):
        pl = [int(x) for x in g["placements"][k]]
        rep = S.simulate(gg, topo, pl)
        assert rep.makespan_seconds == g["makespan"][k]
        assert rep.per_device_busy_seconds == list(g["busy"][k])
        peaks, ok = S.check_memory(gg, topo, pl)
        assert peaks == list(g["peak"][k]) and ok == bool(g["feasible"][k])
        m = S.measure(gg, topo, pl)
        assert m == (g["makespan"][k] if g["feasible"][k] else S.INFEASIBLE)
    with pytest.raises(ValueError):
        S.measure(gg, topo, pl, steps=1)


def test_empty_batch_and_graph_cache():
    gg, topo, _, _ = cfg("C1")
    a = S.device_graph(gg, topo)
    assert S.device_graph(gg, topo) is a
    out = S.simulate_batch(gg, topo, np.zeros((0, gg.num_groups), np.uint8))
    assert out["makespan"].numel() == 0
    torch.cuda.synchronize()
