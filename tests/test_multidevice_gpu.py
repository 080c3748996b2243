"""K-sharded training through the library's own NCCL binding and the
single-process multi-device runner.

The round's GPU box has one B200, so:
* NCCL itself runs with one rank (``dp_comm_init_rank`` / ``ncclCommInitAll``
  over [0]): the exchange-record pack/unpack, the collectives on the step's
  stream and their CUDA-graph capture all execute, and the training log must
  stay byte-identical to the reference's;
* the single-process runner's G-rank orchestration (phases interleaved across
  ranks, collectives between them, one captured graph per update) runs with
  every rank on cuda:0 (parallel.LocalGroup), against the reference's
  single-process train() — byte-identical log, parameters to 1e-12.
"""

import numpy as np
import pytest
import torch

from fixtures import cfg, train_golden, PARAM_RTOL
import paper_1706_04972_b200 as dp
from paper_1706_04972_b200 import parallel, trainer

pytestmark = pytest.mark.gpu


def _check(res, g):
    assert dp.log_to_csv(res.log, include_wall=False) == g["csv"]
    if len(g["best_placement"]):
        assert res.best_placement == [int(x) for x in g["best_placement"]]
    else:
        assert res.best_placement is None
    assert res.store_versions == int(g["store_versions"])
    rel = np.linalg.norm(res.final_params - g["final_params"]) / np.linalg.norm(g["final_params"])
    assert rel < PARAM_RTOL, rel


def test_nccl_binding_loads():
    v = parallel.nccl_version()
    assert v >= 20900  # stream-capturable collectives


@pytest.mark.parametrize("name", ["C1", "C3tight", "C1noise"])
def test_single_rank_nccl_exchange_captured_matches_reference(name):
    gg, topo, _, _ = cfg(name.replace("noise", ""))
    g = train_golden(name)
    config = dp.TrainerConfig(**g["cfg"])
    task = trainer._make_task(gg, topo, config)
    store = dp.ParameterStore(task.template.to_flat(), max_steps=config.total_updates + 1)
    (x,) = parallel.NcclExchange.init_all([torch.cuda.current_device()])
    seq = np.random.SeedSequence(config.seed).spawn(1)[0]
    ctl = trainer.DeviceController(task, store, seq, 0, world=(0, 1, x))
    assert ctl.exchanged and ctl.xchg.capturable
    r = trainer.run_controller(0, store, task, seq, ctl=ctl)
    assert ctl._graph is not None  # the update incl. the NCCL calls was graph-captured
    rows = sorted(r.rows, key=lambda q: (q.controller_id, q.update_index))
    assert dp.log_to_csv(rows, include_wall=False) == g["csv"]
    rel = np.linalg.norm(store.snapshot()[0] - g["final_params"]) / np.linalg.norm(g["final_params"])
    assert rel < PARAM_RTOL


@pytest.mark.parametrize("name,G", [("C1", 2), ("C3tight", 2), ("C3tight", 4), ("C1noise", 2)])
def test_single_process_multi_rank_train_matches_reference(name, G):
    gg, topo, _, _ = cfg(name.replace("noise", ""))
    g = train_golden(name)
    d = torch.cuda.current_device()
    res = dp.train(gg, topo, dp.TrainerConfig(**g["cfg"], devices=(d,) * G))
    _check(res, g)
    assert res.sampling["uncertified_samples"] == 0


def test_multi_device_runner_nccl_group_one_device():
    """The distinct-device path (ncclCommInitAll + group-wrapped collectives +
    per-device graph capture) with the one device this box has."""
    gg, topo, _, _ = cfg("C3tight")
    g = train_golden("C3tight")
    config = dp.TrainerConfig(**g["cfg"])
    task = trainer._make_task(gg, topo, config)
    seq = np.random.SeedSequence(config.seed).spawn(1)[0]
    runner = trainer.MultiDeviceRunner(task, config, [torch.cuda.current_device()], seq)
    assert isinstance(runner.comm, parallel.NcclGroup)
    res = runner.result(runner.train(config.total_updates))
    assert runner._graphs is not None
    _check(res, g)


def test_default_train_uses_visible_devices():
    gg, topo, _, _ = cfg("C1")
    g = train_golden("C1")
    assert trainer._auto_devices(dp.TrainerConfig(**g["cfg"]))[0] == torch.cuda.current_device()
    _check(dp.train(gg, topo, dp.TrainerConfig(**g["cfg"])), g)
