"""f4 on the device: dp_group_features (csrc/features.cu) builds the group-edge
CSR, out_bytes and the policy's GroupFeatures of paper-scale graphs; they must
equal the reference's GroupedGraph / GroupFeatures.from_grouped (goldens in
tests/golden/ingest_*.npz; shape entries within 1 ulp of glibc log1p)."""

import numpy as np
import pytest

from paper_1706_04972_b200 import graph as G
from paper_1706_04972_b200 import ingest as I
from paper_1706_04972_b200.policy import EmbeddingSpec, GroupFeatures
from test_ingest import NAMES, check_features, load

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", NAMES)
def test_device_ingest_matches_reference(name):
    g, a = load(name)
    ga, feats = I.ingest(g)
    parts = [tuple(p) for p in ga.parts]
    pp, po = a["part_ptr"], a["part_ops"]
    assert parts == [tuple(int(x) for x in po[pp[i]:pp[i + 1]]) for i in range(len(pp) - 1)]
    assert ga.topo == a["topo"].tolist()
    src = np.repeat(np.arange(ga.num_groups), np.diff(ga.edge_off))
    assert src.tolist() == a["ge_src"].tolist()
    assert ga.edge_dst.tolist() == a["ge_dst"].tolist()
    assert ga.edge_bytes.tolist() == a["ge_bytes"].tolist()
    assert ga.out_bytes.tolist() == a["group_out_bytes"].tolist()
    assert ga.cost.tolist() == a["group_cost"].tolist()
    assert ga.param_bytes.tolist() == a["group_param"].tolist()
    check_features(feats, a, shape_ulps=1)


def test_device_features_equal_host_features_with_unknown_types():
    """A spec built from another graph: types missing from its vocabulary map to
    the unknown row but keep their name order (pkg/policy.py:63-64, 105-107)."""
    g, a = load("rnnlm_L2S20")
    fixed = G.split_cyclic_groups(g)
    gg = G.coalesce_sole_consumers(fixed)
    names = sorted({op.op_type for op in g.ops})
    spec = EmbeddingSpec({t: i for i, t in enumerate(names[::2])}, shape_slots=11, adjacency_slots=7)
    ga = I.grouped_arrays(fixed, [grp.members for grp in gg.groups], spec)
    got = I.features_for(ga)
    want = GroupFeatures.from_grouped(gg, spec)
    assert list(got.order) == list(want.order)
    for x, y in zip(got.type_indices, want.type_indices):
        assert np.asarray(x).tolist() == np.asarray(y).tolist()
    assert np.array_equal(got.adj_blocks, want.adj_blocks)
    ulp = np.abs(np.asarray(got.shape_blocks).view(np.int64) - np.asarray(want.shape_blocks).view(np.int64))
    assert int(ulp.max()) <= 1


def test_device_ingest_rejects_cyclic_grouping():
    g, _ = load("rnnlm_L2S20")
    with pytest.raises(ValueError, match="cycle between groups"):
        I.ingest(g, split=False)
