"""World-size-2 (gloo, CPU) test of the K-sharded exchange used by the multi-GPU
controller (paper_1706_04972_b200/parallel.py).

Each rank samples ONLY its shard (advancing the reference PCG64 stream to draw
k_offset*T), scores and differentiates it with the CPU oracle, then uses the
product's Exchange to all-gather scores/placements and all-reduce the
gradient.  The result must equal the reference's single-process update
(tests/golden/train_C1.npz): placements bit-exact, gradient to 1e-10.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1706_04972_b200.parallel import Exchange, draw_index, shard


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, size, port, out_q):
    import sys

    here = os.path.dirname(os.path.abspath(__file__))
    sys.path.insert(0, here)
    sys.path.insert(0, os.path.dirname(here))
    from fixtures import cfg, train_golden
    from oracle import policy as opol
    from oracle import trainer as otr
    from oracle.sim import OracleGraph

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=size)
    try:
        gg, topo, _, _ = cfg("C1")
        g = train_golden("C1")
        K = g["cfg"]["k"]
        T = gg.num_groups
        k0, kl = shard(K, rank, size)
        dims = otr.dims_for(gg, topo, {})
        feats = opol.features(gg, opol.vocab_of(gg))
        pol = opol.Policy(opol.init_flat(dims, 0), dims, feats)
        rng = np.random.default_rng(np.random.SeedSequence(0).spawn(1)[0].spawn(2)[0])
        rng.bit_generator.advance(draw_index(0, k0, 0, K, T))
        draws = [pol.sample(rng) for _ in range(kl)]
        rep = OracleGraph(gg, topo).simulate([d[0] for d in draws])
        order = np.asarray(gg.topo)
        ch_local = torch.tensor(np.array([np.asarray(d[0])[order] for d in draws], np.uint8))
        mk_local = torch.tensor(rep["makespan"])
        fe_local = torch.tensor(rep["feasible"])
        ex = Exchange(None)
        mk = ex.all_gather(torch.zeros(K, dtype=torch.float64), mk_local)
        fe = ex.all_gather(torch.zeros(K, dtype=torch.uint8), fe_local)
        ch = ex.all_gather(torch.zeros(K, T, dtype=torch.uint8), ch_local)
        # replicated epilogue (reference order) on the gathered scores
        fail = otr.failing_signal(gg, topo)
        R = [otr.reward(float(m) if f else otr.INF, fail) for m, f in zip(mk.numpy(), fe.numpy())]
        b = fail
        grad = np.zeros(dims.n_params)
        for i, d in enumerate(draws):
            grad += (R[k0 + i] - b) * pol.grad(d[0], d[2])
        gt = torch.tensor(grad)
        ex.all_reduce_sum(gt)
        out_q.put((rank, ch.numpy(), mk.numpy(), (gt / K).numpy(), 0.9 * b + 0.1 * float(np.mean(R))))
    finally:
        dist.destroy_process_group()


def test_shard_bounds():
    assert shard(256, 0, 8) == (0, 32) and shard(256, 7, 8) == (224, 32)
    with pytest.raises(ValueError):
        shard(10, 0, 3)
    assert draw_index(2, 3, 5, K=8, T=100) == 2 * 800 + 300 + 5


def test_two_rank_exchange_matches_single_process_reference():
    from fixtures import cfg, train_golden

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(2):
        r = q.get(timeout=300)
        res[r[0]] = r
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    gg, topo, _, _ = cfg("C1")
    g = train_golden("C1")
    order = np.asarray(gg.topo)
    ref_by_rank = g["placements"][0][:, order]
    for rank in (0, 1):
        _, ch, mk, grad, base = res[rank]
        assert np.array_equal(ch, ref_by_rank)                   # both ranks hold all K placements
        assert np.array_equal(mk, g["measure"][0])                # and all K scores
        rel = np.linalg.norm(grad - g["grads"][0]) / np.linalg.norm(g["grads"][0])
        assert rel < 1e-10
        assert base == float(g["baseline_before"][1])              # replicated baseline, bit-exact
    assert np.array_equal(res[0][3], res[1][3])                     # replicated gradient
