"""f4 graph ingestion: the reference generators' cyclic
co-location seeds made acyclic, and the group arrays / policy features of the
resulting paper-scale graphs.

Goldens (tests/golden/ingest_*.npz, ``make_golden.py ingest``) hold the op
graph and its shipped manual groups (``pkg/generators.py:132-150``), the split
seeds (the input under test), and the REFERENCE's own coalescing,
GroupedGraph (``pkg/graph.py:183-338``) and GroupFeatures.from_grouped
(``pkg/policy.py:97-114``) on that input."""

import math
import os

import numpy as np
import pytest

from paper_1706_04972_b200 import graph as G
from paper_1706_04972_b200.policy import EmbeddingSpec, GroupFeatures

HERE = os.path.dirname(os.path.abspath(__file__))
NAMES = ["rnnlm_L2S20", "nmt_L4S40"]


def load(name):
    a = dict(np.load(os.path.join(HERE, "golden", f"ingest_{name}.npz"), allow_pickle=False))
    types = [str(t) for t in a["types"]]
    sp, dims = a["shape_ptr"], a["shape_dims"]
    ops = [G.Operation(i, f"op{i}", types[int(a["op_type"][i])], float(a["op_cost"][i]),
                       tuple(int(x) for x in dims[sp[i]:sp[i + 1]]), int(a["op_param"][i]))
           for i in range(len(a["op_type"]))]
    edges = [G.Edge(int(s), int(d), int(b)) for s, d, b in zip(a["edge_src"], a["edge_dst"], a["edge_bytes"])]
    mp, mo = a["manual_ptr"], a["manual_ops"]
    manual = [[int(x) for x in mo[mp[i]:mp[i + 1]]] for i in range(len(mp) - 1)]
    return G.ComputationGraph(ops, edges, manual), a


def groups_of(ptr, ops):
    return [tuple(int(x) for x in ops[ptr[i]:ptr[i + 1]]) for i in range(len(ptr) - 1)]


@pytest.mark.parametrize("name", NAMES)
def test_shipped_manual_groups_are_cyclic(name):
    g, _ = load(name)
    with pytest.raises(G.GraphError, match="cycle between groups"):
        G.coalesce_sole_consumers(g)


@pytest.mark.parametrize("name", NAMES)
def test_split_cyclic_groups(name):
    g, a = load(name)
    fixed = G.split_cyclic_groups(g)
    assert sorted(tuple(x) for x in fixed.manual_groups) == sorted(groups_of(a["split_ptr"], a["split_ops"]))
    # every split group lies inside one shipped group, and a shipped unit
    # becomes at most two groups: its forward chain and its backward mirror
    # (ops named .../grad_*), or stays whole when no cycle runs through it
    owner = {}
    for gi, grp in enumerate(g.manual_groups):
        for i in grp:
            owner[i] = gi
    grad = a["op_name_grad"]
    pieces = {}
    for grp in fixed.manual_groups:
        assert len({owner[i] for i in grp}) == 1
        pieces.setdefault(owner[grp[0]], []).append(grp)
    for gi, ps in pieces.items():
        assert len(ps) <= 2
        if len(ps) == 2:
            assert sorted(len({bool(grad[i]) for i in p}) for p in ps) == [1, 1]
    # the quotient is acyclic: GroupedGraph accepts seeds + singletons
    covered = {i for grp in fixed.manual_groups for i in grp}
    G.GroupedGraph(fixed, [tuple(x) for x in fixed.manual_groups] + [(i,) for i in range(g.num_ops) if i not in covered])


@pytest.mark.parametrize("name", NAMES)
def test_host_grouping_and_features_match_reference(name):
    g, a = load(name)
    fixed = G.split_cyclic_groups(g)
    parts = G.coalesce_partition(fixed)
    assert sorted(parts) == sorted(groups_of(a["part_ptr"], a["part_ops"]))
    gg = G.GroupedGraph(fixed, parts)
    assert list(gg.topo) == a["topo"].tolist()
    assert [(e.src, e.dst, e.tensor_bytes) for e in gg.group_edges] == list(
        zip(a["ge_src"].tolist(), a["ge_dst"].tolist(), a["ge_bytes"].tolist()))
    assert [grp.compute_cost for grp in gg.groups] == a["group_cost"].tolist()
    assert [grp.out_bytes for grp in gg.groups] == a["group_out_bytes"].tolist()
    spec = EmbeddingSpec.build([gg])
    assert sorted(spec.type_vocab, key=spec.type_vocab.get) == [str(v) for v in a["vocab"]]
    f = GroupFeatures.from_grouped(gg, spec)
    check_features(f, a, shape_ulps=0)


def check_features(f, a, shape_ulps):
    assert list(f.order) == a["topo"].tolist()
    off = a["f_type_off"]
    for t, ix in enumerate(f.type_indices):
        assert np.asarray(ix).tolist() == a["f_type_idx"][off[t]:off[t + 1]].tolist(), t
    adj = np.zeros_like(np.asarray(f.adj_blocks))
    adj[a["f_adj_t"], a["f_adj_s"].astype(np.int64)] = 1.0
    assert np.array_equal(np.asarray(f.adj_blocks), adj)
    got, want = np.asarray(f.shape_blocks), a["f_shape"]
    if shape_ulps == 0:
        assert np.array_equal(got, want)
    else:
        ulp = np.abs(got.view(np.int64) - want.view(np.int64))
        assert int(ulp.max()) <= shape_ulps
