"""f1 (asynchronous multi-controller training over one device-resident store)
and C4 (several independent tasks advanced together on their own streams)."""

import numpy as np
import pytest

from fixtures import cfg, train_golden, PARAM_RTOL
from oracle import trainer as otr
import paper_1706_04972_b200 as dp

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name,C,K,U", [("C1", 3, 8, 3), ("C3tight", 2, 8, 3)])
def test_multi_controller_round_schedule_matches_oracle(name, C, K, U):
    """C controllers share the store; every round they sample from one version
    and apply in controller order (oracle.trainer.run_multi)."""
    gg, topo, _, _ = cfg(name)
    d = dict(k=K, total_updates=U, seed=5, controllers=C, success_only_after=2 if name == "C3tight" else 5000)
    res = dp.train(gg, topo, dp.TrainerConfig(**d))
    want = otr.run_multi(gg, topo, d)
    assert dp.log_to_csv(res.log, include_wall=False) == otr.csv_of(want["rows"])
    assert res.store_versions == want["versions"]
    rel = np.linalg.norm(res.final_params - want["final"]) / np.linalg.norm(want["final"])
    assert rel < PARAM_RTOL
    # properties of any admissible interleaving: one row per (controller, update),
    # versions never decrease per controller, best_R monotone
    assert len(res.log) == C * U
    for c in range(C):
        rows = [r for r in res.log if r.controller_id == c]
        assert [r.update_index for r in rows] == list(range(U))
        assert all(a.store_version <= b.store_version for a, b in zip(rows, rows[1:]))
        assert all(a.best_r >= b.best_r for a, b in zip(rows, rows[1:]))
    if want["best_placement"] is not None:
        assert res.best_placement == want["best_placement"]


def test_train_many_concurrent_equals_each_run_alone():
    """C4-style mixed batch: two tasks with equal update counts share one graph
    replay per round (own streams); each equals the reference run alone."""
    g1, t1, _, _ = cfg("C1")
    a, b = train_golden("C1"), train_golden("C1noise")
    ra, rb = dp.train_many([(g1, t1, dp.TrainerConfig(**a["cfg"])), (g1, t1, dp.TrainerConfig(**b["cfg"]))])
    for res, g in ((ra, a), (rb, b)):
        assert dp.log_to_csv(res.log, include_wall=False) == g["csv"]
        rel = np.linalg.norm(res.final_params - g["final_params"]) / np.linalg.norm(g["final_params"])
        assert rel < PARAM_RTOL


def test_train_many_mixed_graphs_and_lengths():
    g1, t1, _, _ = cfg("C1")
    g2, t2, _, _ = cfg("C2")
    a, b = train_golden("C1"), train_golden("C2")
    ra, rb = dp.train_many([(g1, t1, dp.TrainerConfig(**a["cfg"])), (g2, t2, dp.TrainerConfig(**b["cfg"]))])
    assert dp.log_to_csv(ra.log, include_wall=False) == a["csv"]
    assert dp.log_to_csv(rb.log, include_wall=False) == b["csv"]
