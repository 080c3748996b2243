"""f3: brute-force and random-search baselines as batched K-sim fan-outs,
against the reference's own results (tests/golden/baselines.npz)."""

import itertools

import numpy as np
import pytest

from fixtures import baseline_cases, cfg
import paper_1706_04972_b200 as dp

pytestmark = pytest.mark.gpu


def test_brute_force_matches_reference():
    cases, _ = baseline_cases()
    n_nofeas = 0
    for i, (gg, topo, bf, mk, _b, _rs) in enumerate(cases):
        if bf is None:
            n_nofeas += 1
            with pytest.raises(dp.NoFeasiblePlacement):
                dp.brute_force(gg, topo)
        else:
            pl, got = dp.brute_force(gg, topo)
            assert pl == bf, i
            assert got == mk, i
    assert n_nofeas >= 2


def test_random_search_matches_reference():
    cases, c1_rs = baseline_cases()
    for i, (gg, topo, _bf, _mk, budget, rs) in enumerate(cases):
        assert dp.place_random_search(gg, topo, budget=budget, seed=i) == rs, i
    gg, topo, _, _ = cfg("C1")
    assert dp.place_random_search(gg, topo, budget=300, seed=11) == c1_rs


def test_brute_force_multi_batch_ties_resolve_lexicographically():
    """A search space of several 64K batches where every placement ties: the
    answer must be placement 0...0 (itertools.product order)."""
    ops = [dp.Operation(i, f"op{i}", "t", 0.0, (1,), 0) for i in range(18)]
    gg = dp.singleton_groups(dp.ComputationGraph(ops, []))
    topo = dp.default_topology(1)
    pl, mk = dp.brute_force(gg, topo)
    assert pl == [0] * 18 and mk == 0.0


def test_brute_force_errors():
    gg, topo, _, _ = cfg("C1")
    with pytest.raises(dp.SearchSpaceTooLarge):
        dp.brute_force(gg, topo)
    with pytest.raises(ValueError):
        dp.place_random_search(gg, topo, budget=0)
    assert dp.place_single(gg, topo, 1) == [1] * gg.num_groups
    with pytest.raises(ValueError):
        dp.place_single(gg, topo, 7)
