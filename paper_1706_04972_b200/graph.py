"""Input data model of the placement hot path: op graphs and co-location groups.

The hot path consumes a *grouped* graph: per-group
compute cost, resident bytes, deduplicated group edges and a deterministic
topological rank.  This module rebuilds those objects with the same field
names and semantics as the reference so either side's objects can be passed to
the simulator / policy / trainer entry points (duck typing):

* ``ComputationGraph``   — reference ``pkg/graph.py:66-161``
* ``GroupedGraph``       — reference ``pkg/graph.py:183-274`` (group ids ordered
  by smallest member op, fsum costs, out_bytes counting intra-group edges,
  (src, dst)-sorted deduplicated edges, Kahn topo order with a min-gid heap)
* ``coalesce_sole_consumers`` — reference ``pkg/graph.py:282-338``

Graph construction is one-time host preprocessing (out of the per-step hot
path); the device upload of the resulting arrays lives in
:mod:`paper_1706_04972_b200.simulator`.
"""

from __future__ import annotations

import heapq
import math
from collections import Counter
from dataclasses import dataclass, field


class GraphError(ValueError):
    """Schema violation in a graph (reference ``pkg/graph.py:22``)."""


class CycleError(GraphError):
    def __init__(self, message: str, cycle: list[int]):
        super().__init__(message)
        self.cycle = cycle


@dataclass(frozen=True)
class Operation:
    id: int
    name: str
    op_type: str
    compute_cost: float
    output_shape: tuple = ()
    param_bytes: int = 0

    def output_elems(self) -> int:
        return math.prod(self.output_shape) if self.output_shape else 0


@dataclass(frozen=True)
class Edge:
    src: int
    dst: int
    tensor_bytes: int


def _kahn_min_heap(n: int, succ: list[list[int]]) -> list[int]:
    """Topological order, smallest ready id first (reference graph.py:127-143, 252-266)."""
    indeg = [0] * n
    for outs in succ:
        for w in outs:
            indeg[w] += 1
    heap = [v for v in range(n) if indeg[v] == 0]
    heapq.heapify(heap)
    order = []
    while heap:
        v = heapq.heappop(heap)
        order.append(v)
        for w in succ[v]:
            indeg[w] -= 1
            if indeg[w] == 0:
                heapq.heappush(heap, w)
    return order


class ComputationGraph:
    """Validated op DAG (reference ``pkg/graph.py:66-161``)."""

    def __init__(self, ops, edges, manual_groups=None):
        self.ops = list(ops)
        self.edges = list(edges)
        self.manual_groups = [list(g) for g in (manual_groups or [])]
        m = len(self.ops)
        for i, op in enumerate(self.ops):
            if op.id != i:
                raise GraphError(f"op ids must be dense 0..{m - 1} in order; position {i} has id {op.id}")
            if not (op.compute_cost >= 0.0 and math.isfinite(op.compute_cost)):
                raise GraphError(f"op {op.id} ({op.name}): compute_cost must be finite and >= 0")
            if op.param_bytes < 0:
                raise GraphError(f"op {op.id} ({op.name}): param_bytes must be >= 0")
            if any(d < 1 for d in op.output_shape):
                raise GraphError(f"op {op.id} ({op.name}): output_shape dims must be >= 1")
        for e in self.edges:
            if not (0 <= e.src < m and 0 <= e.dst < m):
                raise GraphError(f"edge {e.src}->{e.dst}: dangling endpoint")
            if e.src == e.dst:
                raise GraphError(f"self-edge on op {e.src}")
            if e.tensor_bytes < 0:
                raise GraphError(f"edge {e.src}->{e.dst}: tensor_bytes must be >= 0")
        seen: set[int] = set()
        for grp in self.manual_groups:
            for i in grp:
                if not (0 <= i < m):
                    raise GraphError(f"manual_groups references unknown op id {i}")
                if i in seen:
                    raise GraphError(f"manual_groups overlap on op id {i}")
                seen.add(i)
        self.out_ids = [[] for _ in range(m)]
        self.in_ids = [[] for _ in range(m)]
        for e in self.edges:
            self.out_ids[e.src].append(e.dst)
            self.in_ids[e.dst].append(e.src)
        self.topo_order = _kahn_min_heap(m, self.out_ids)
        if len(self.topo_order) < m:
            left = sorted(set(range(m)) - set(self.topo_order))
            raise CycleError("graph contains a cycle", left)

    @property
    def num_ops(self) -> int:
        return len(self.ops)

    def total_compute_cost(self) -> float:
        return math.fsum(op.compute_cost for op in self.ops)

    def total_param_bytes(self) -> int:
        return sum(op.param_bytes for op in self.ops)


@dataclass(frozen=True)
class Group:
    id: int
    members: tuple
    compute_cost: float
    param_bytes: int
    out_bytes: int
    type_counts: dict = field(hash=False, compare=False, default_factory=dict)


@dataclass(frozen=True)
class GroupEdge:
    src: int
    dst: int
    tensor_bytes: int


class GroupedGraph:
    """Co-location groups over a ComputationGraph (reference ``pkg/graph.py:183-274``)."""

    def __init__(self, graph: ComputationGraph, partition):
        self.graph = graph
        parts = sorted((tuple(sorted(p)) for p in partition), key=lambda p: p[0])
        member_of = [-1] * graph.num_ops
        for gid, members in enumerate(parts):
            for op_id in members:
                member_of[op_id] = gid
        if min(member_of, default=0) < 0:
            raise GraphError("partition does not cover every op")
        self.membership = member_of
        out_bytes = [0] * len(parts)
        cross: dict[tuple[int, int], int] = {}
        for e in graph.edges:
            gs, gd = member_of[e.src], member_of[e.dst]
            out_bytes[gs] += e.tensor_bytes
            if gs != gd:
                cross[(gs, gd)] = cross.get((gs, gd), 0) + e.tensor_bytes
        ops = graph.ops
        self.groups = [
            Group(gid, members,
                  math.fsum(ops[i].compute_cost for i in members),
                  sum(ops[i].param_bytes for i in members),
                  out_bytes[gid],
                  dict(Counter(ops[i].op_type for i in members)))
            for gid, members in enumerate(parts)
        ]
        self.group_edges = [GroupEdge(s, d, b) for (s, d), b in sorted(cross.items())]
        n = len(self.groups)
        self.out_groups = [[] for _ in range(n)]
        self.in_groups = [[] for _ in range(n)]
        for ge in self.group_edges:
            self.out_groups[ge.src].append(ge.dst)
            self.in_groups[ge.dst].append(ge.src)
        self.topo = _kahn_min_heap(n, self.out_groups)
        if len(self.topo) < n:
            raise GraphError(
                "grouping creates a cycle between groups; manual_groups must "
                "not contain two ops connected through an op outside the group")
        self.topo_rank = [0] * n
        for r, gid in enumerate(self.topo):
            self.topo_rank[gid] = r

    @property
    def num_groups(self) -> int:
        return len(self.groups)

    def total_compute_cost(self) -> float:
        return math.fsum(g.compute_cost for g in self.groups)

    def output_elem_counts(self, gid: int) -> list[int]:
        counts = (self.graph.ops[i].output_elems() for i in self.groups[gid].members)
        return [c for c in counts if c > 0]


def topo_order(gg) -> list[int]:
    return list(gg.topo)


def singleton_groups(graph: ComputationGraph) -> GroupedGraph:
    return GroupedGraph(graph, [(i,) for i in range(graph.num_ops)])


def coalesce_sole_consumers(graph: ComputationGraph) -> GroupedGraph:
    """Manual seeds, then merge any group feeding exactly one other group until a
    fixed point; sweeps visit groups by ascending representative id and the
    smaller representative survives (reference ``pkg/graph.py:282-338``)."""
    return GroupedGraph(graph, coalesce_partition(graph))


def coalesce_partition(graph) -> list:
    """The member tuples of :func:`coalesce_sole_consumers` (reference
    ``_coalesce_partition``, ``pkg/graph.py:282-332``); duck typed over the
    reference's ComputationGraph as well."""
    rep = list(range(len(graph.ops)))

    def root(x):
        while rep[x] != x:
            rep[x] = rep[rep[x]]
            x = rep[x]
        return x

    members = {i: [i] for i in range(len(graph.ops))}
    for seed in graph.manual_groups:
        if len(seed) < 2:
            continue
        keep = min(root(i) for i in seed)
        for i in seed:
            r = root(i)
            if r != keep:
                rep[r] = keep
                members[keep].extend(members.pop(r))
    changed = True
    while changed:
        changed = False
        for r in sorted(members):
            if r not in members:
                continue
            consumers = {root(d) for op in members[r] for d in graph.out_ids[op]} - {r}
            if len(consumers) != 1:
                continue
            other = consumers.pop()
            keep, drop = (r, other) if r < other else (other, r)
            rep[drop] = keep
            members[keep].extend(members.pop(drop))
            changed = True
    return [tuple(sorted(v)) for v in members.values()]


def split_cyclic_groups(graph):
    """Co-location seeds that keep the group graph acyclic.

    The reference generators seed one manual group per model unit holding its
    forward chain AND its backward mirror (``pkg/generators.py:132-143``);
    units linked forward (src -> dst) and backward (dst -> src,
    ``pkg/generators.py:146-150``) then form a cycle between groups, and
    ``GroupedGraph`` rejects the grouping (``pkg/graph.py:266-272``).  This
    splits every manual group into the runs its members form in a
    group-greedy topological order of the ops (Kahn; the current group keeps
    going while it has a ready op, else the smallest ready op id starts the
    next run).  Runs are contiguous in one topological order, so every edge
    between runs points forward: the quotient is acyclic.  A unit's forward
    chain and backward mirror become two groups; an already-acyclic grouping
    whose groups are convex keeps each group whole.

    Accepts the reference's ``ComputationGraph`` or this package's (duck typed:
    ``ops``, ``edges``, ``manual_groups``, ``out_ids``, ``in_ids``) and returns
    the same class with the new ``manual_groups``."""
    m = len(graph.ops)
    grp = [-1] * m
    for g, members in enumerate(graph.manual_groups):
        for i in members:
            grp[i] = g
    indeg = [len(x) for x in graph.in_ids]
    ready = [v for v in range(m) if indeg[v] == 0]
    heapq.heapify(ready)
    ready_of: dict[int, list[int]] = {}
    for v in ready:
        if grp[v] >= 0:
            heapq.heappush(ready_of.setdefault(grp[v], []), v)
    done = [False] * m
    runs: list[list[int]] = []
    cur, run = -1, None
    placed = 0
    while placed < m:
        v = -1
        if cur >= 0:
            h = ready_of.get(cur)
            while h and done[h[0]]:
                heapq.heappop(h)
            if h:
                v = heapq.heappop(h)
        if v < 0:
            while done[ready[0]]:
                heapq.heappop(ready)
            v = heapq.heappop(ready)
            if grp[v] != cur or grp[v] < 0:
                cur = grp[v]
                run = [] if cur >= 0 else None
                if run is not None:
                    runs.append(run)
        done[v] = True
        placed += 1
        if run is not None:
            run.append(v)
        for w in graph.out_ids[v]:
            indeg[w] -= 1
            if indeg[w] == 0:
                heapq.heappush(ready, w)
                if grp[w] >= 0:
                    heapq.heappush(ready_of.setdefault(grp[w], []), w)
    new_groups = [sorted(r) for r in runs if len(r) > 1]
    return type(graph)(graph.ops, graph.edges, new_groups)
