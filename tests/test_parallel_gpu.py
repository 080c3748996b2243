"""Multi-rank K-sharded training on the device path.

The round's GPU box has one B200, so the two ranks share cuda:0 and exchange
through gloo (host-staged; the same Exchange code NCCL uses on 8 GPUs).  Each
rank samples, scores and differentiates only its K/2 shard; the all-gathered
scores and all-reduced gradient must reproduce the reference's single-process
train() run: byte-identical log, same best placement, parameters to 1e-12.
"""

import os
import socket
import subprocess
import sys
import json

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, size, port, name, q):
    import torch.distributed as dist

    here = os.path.dirname(os.path.abspath(__file__))
    sys.path.insert(0, here)
    sys.path.insert(0, os.path.dirname(here))
    from fixtures import cfg, train_golden

    import paper_1706_04972_b200 as dp

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=size)
    try:
        gg, topo, _, _ = cfg(name)
        g = train_golden(name)
        res = dp.train(gg, topo, dp.TrainerConfig(**g["cfg"]), group=dist.group.WORLD)
        q.put((rank, dp.log_to_csv(res.log, include_wall=False), res.best_placement, res.final_params,
               res.store_versions))
    except Exception as ex:  # pragma: no cover - surfaced by the parent
        q.put((rank, repr(ex), None, None, None))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name,size", [("C1", 2), ("C3tight", 2), ("C3tight", 4)])
def test_sharded_train_matches_single_process_reference(name, size):
    from fixtures import PARAM_RTOL, train_golden

    g = train_golden(name)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, size, port, name, q)) for r in range(size)]
    for p in procs:
        p.start()
    outs = sorted([q.get(timeout=300) for _ in procs], key=lambda o: o[0])
    for p in procs:
        p.join(timeout=60)
    for rank, csv, best, final, versions in outs:
        assert csv == g["csv"], (rank, csv)
        if len(g["best_placement"]):
            assert best == [int(x) for x in g["best_placement"]]
        assert versions == int(g["store_versions"])
        rel = np.linalg.norm(final - g["final_params"]) / np.linalg.norm(g["final_params"])
        assert rel < PARAM_RTOL, (rank, rel)


def test_bench_multi_rank_line():
    """bench.py under torchrun (2 ranks on one GPU, gloo): one JSON line, K sharded."""
    env = dict(os.environ, DP_DIST_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "bench.py", "--gpus", "2",
           "--steps", "3", "--warmup", "3", "--config", "C1", "--profile-phases", "1"]
    out = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["config"]["global_k"] == 2 * d["config"]["k_per_gpu"]
    assert d["value"] > 0 and d["e2e"]["value"] > 0
