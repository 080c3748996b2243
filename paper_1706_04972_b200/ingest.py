"""Graph ingestion for paper-scale op graphs.

Two pieces in front of the hot path:

* :func:`split_cyclic_groups` (host, :mod:`.graph`) makes the reference
  generators' co-location seeds acyclic (``pkg/generators.py:132-150`` puts a
  unit's forward chain and backward mirror in one group, so linked units form
  a cycle between groups and ``GroupedGraph`` rejects them,
  ``pkg/graph.py:266-272``).
* :func:`grouped_arrays` builds, on the GPU (``dp_group_features``,
  ``csrc/features.cu``), what the reference computes per group in Python
  loops: the deduplicated group-edge CSR with summed bytes and out_bytes
  (``pkg/graph.py:183-238``) and the policy's GroupFeatures — type multiset,
  shape block, adjacency multi-hot (``pkg/policy.py:97-114``).  The host adds
  the exact ``math.fsum`` group costs and the Kahn min-heap topological order
  (``pkg/graph.py:252-266``) over the returned CSR, then orders the feature
  rows by rank.

:func:`features_for` returns a :class:`~.policy.GroupFeatures` equal to the
reference's ``GroupFeatures.from_grouped`` (shape entries within one ulp of
glibc ``log1p``) without constructing per-group Python objects.
"""

from __future__ import annotations

import ctypes
import heapq
import math
from dataclasses import dataclass

import numpy as np

from .graph import split_cyclic_groups  # noqa: F401  (re-export: the f4 host fix)
from .policy import EmbeddingSpec, GroupFeatures


def _hp(a):
    return a.ctypes.data_as(ctypes.c_void_p)


@dataclass
class GroupedArrays:
    """Group-level arrays of a grouped op graph, indexed by group id
    (groups ordered by smallest member op id, as ``GroupedGraph``)."""

    parts: list          # member tuples
    membership: np.ndarray  # op -> group id
    cost: np.ndarray     # fsum of member compute costs
    param_bytes: np.ndarray
    out_bytes: np.ndarray
    edge_off: np.ndarray  # CSR over group out-edges (to other groups), by destination id
    edge_dst: np.ndarray
    edge_bytes: np.ndarray
    topo: list           # Kahn order, smallest ready group id first
    type_off: np.ndarray  # by group id
    type_idx: np.ndarray
    shape: np.ndarray     # [G, shape_slots]
    adj: np.ndarray       # [G, adjacency_slots]

    @property
    def num_groups(self) -> int:
        return len(self.parts)

    def in_groups(self) -> list:
        ins = [[] for _ in range(self.num_groups)]
        for s in range(self.num_groups):
            for d in self.edge_dst[self.edge_off[s]:self.edge_off[s + 1]]:
                ins[int(d)].append(s)
        return ins


def _kahn(n, off, dst):
    indeg = np.bincount(dst, minlength=n).astype(np.int64) if len(dst) else np.zeros(n, np.int64)
    heap = [v for v in range(n) if indeg[v] == 0]
    heapq.heapify(heap)
    order = []
    while heap:
        v = heapq.heappop(heap)
        order.append(v)
        for w in dst[off[v]:off[v + 1]]:
            w = int(w)
            indeg[w] -= 1
            if indeg[w] == 0:
                heapq.heappush(heap, w)
    return order


def grouped_arrays(graph, partition, spec: EmbeddingSpec) -> GroupedArrays:
    """Group-level arrays and policy features of ``graph`` under ``partition``
    (iterable of op-id collections covering every op), built on the GPU."""
    from . import _native as nat

    ops = graph.ops
    n = len(ops)
    parts = sorted((tuple(sorted(p)) for p in partition), key=lambda p: p[0])
    G = len(parts)
    member = np.full(n, -1, np.int32)
    for gid, p in enumerate(parts):
        member[list(p)] = gid
    if (member < 0).any():
        raise ValueError("partition does not cover every op")
    names = sorted({op.op_type for op in ops})
    key_of = {t: i for i, t in enumerate(names)}
    op_key = np.array([key_of[op.op_type] for op in ops], np.int32)
    key_to_index = np.array([spec.index_of(t) for t in names], np.int32)
    elems = np.array([op.output_elems() for op in ops], np.int64)
    E = len(graph.edges)
    src = np.array([e.src for e in graph.edges], np.int32)
    dst = np.array([e.dst for e in graph.edges], np.int32)
    byt = np.array([e.tensor_bytes for e in graph.edges], np.int64)
    ss, aslots = spec.shape_slots, spec.adjacency_slots
    type_off = np.zeros(G + 1, np.int32)
    type_idx = np.zeros(n, np.int32)
    shape = np.zeros((G, ss), np.float64)
    adj = np.zeros((G, aslots), np.float64)
    ge_off = np.zeros(G + 1, np.int32)
    ge_dst = np.zeros(max(E, 1), np.int32)
    ge_bytes = np.zeros(max(E, 1), np.int64)
    out_bytes = np.zeros(G, np.int64)
    rc = nat.lib().dp_group_features(n, G, _hp(member), _hp(op_key), len(names), _hp(key_to_index), _hp(elems), E,
                                     _hp(src), _hp(dst), _hp(byt), ss, aslots, _hp(type_off), _hp(type_idx),
                                     _hp(shape), _hp(adj), _hp(ge_off), _hp(ge_dst), _hp(ge_bytes), _hp(out_bytes))
    nat.check(rc, "dp_group_features")
    ne = int(ge_off[G])
    ge_dst, ge_bytes = ge_dst[:ne].copy(), ge_bytes[:ne].copy()
    topo = _kahn(G, ge_off, ge_dst)
    if len(topo) < G:
        raise ValueError("grouping creates a cycle between groups; manual_groups must "
                         "not contain two ops connected through an op outside the group")
    cost = np.array([math.fsum(ops[i].compute_cost for i in p) for p in parts], np.float64)
    param = np.array([sum(ops[i].param_bytes for i in p) for p in parts], np.int64)
    return GroupedArrays(parts, member, cost, param, out_bytes, ge_off, ge_dst, ge_bytes, topo, type_off, type_idx,
                         shape, adj)


def features_for(ga: GroupedArrays) -> GroupFeatures:
    """GroupFeatures (rows in topological order) from device-built arrays."""
    order = list(ga.topo)
    tix = [ga.type_idx[ga.type_off[g]:ga.type_off[g + 1]].astype(np.intp) for g in order]
    return GroupFeatures(order, tix, ga.shape[order].copy(), ga.adj[order].copy())


def ingest(graph, spec: EmbeddingSpec | None = None, split: bool = True):
    """Paper-scale front door: split cyclic co-location seeds, coalesce
    sole consumers (reference ``pkg/graph.py:282-338``), then build the group
    arrays and features on the device.  Returns (GroupedArrays, GroupFeatures)."""
    from .graph import coalesce_partition

    g = split_cyclic_groups(graph) if split else graph
    parts = coalesce_partition(g)
    if spec is None:
        spec = EmbeddingSpec.build([g])
    ga = grouped_arrays(g, parts, spec)
    return ga, features_for(ga)
