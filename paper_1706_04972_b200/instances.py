"""Compact on-disk form of a placement instance (op graph + grouping + topology).

Benchmark and parity instances (SURVEY.md §8(d) configs C1–C5) are built once
from the reference's public constructors and stored as ``.npz`` so that the GPU
box — where the reference does not exist — can rebuild bit-identical
``GroupedGraph`` / ``DeviceTopology`` objects.  Works on reference objects and
on this package's own (duck typed): only public fields are read.
"""

from __future__ import annotations

import numpy as np

from .graph import ComputationGraph, Edge, GroupedGraph, Operation
from .simulator import Device, DeviceTopology


def instance_arrays(gg, topo) -> dict:
    """Serialize a grouped graph (with its op graph) and a topology."""
    g = gg.graph
    types = sorted({op.op_type for op in g.ops})
    tix = {t: i for i, t in enumerate(types)}
    shape_ptr = np.zeros(len(g.ops) + 1, np.int64)
    dims = []
    for i, op in enumerate(g.ops):
        dims.extend(op.output_shape)
        shape_ptr[i + 1] = len(dims)
    part_ptr = np.zeros(gg.num_groups + 1, np.int64)
    part_ops = []
    for gid, grp in enumerate(gg.groups):
        part_ops.extend(grp.members)
        part_ptr[gid + 1] = len(part_ops)
    return dict(
        types=np.array(types),
        op_type=np.array([tix[op.op_type] for op in g.ops], np.int32),
        op_cost=np.array([op.compute_cost for op in g.ops], np.float64),
        op_param=np.array([op.param_bytes for op in g.ops], np.int64),
        shape_ptr=shape_ptr,
        shape_dims=np.array(dims, np.int64),
        edge_src=np.array([e.src for e in g.edges], np.int32),
        edge_dst=np.array([e.dst for e in g.edges], np.int32),
        edge_bytes=np.array([e.tensor_bytes for e in g.edges], np.int64),
        part_ptr=part_ptr,
        part_ops=np.array(part_ops, np.int32),
        dev_kind=np.array([1 if d.kind == "gpu" else 0 for d in topo.devices], np.int8),
        dev_rate=np.array([d.compute_rate for d in topo.devices], np.float64),
        dev_mem=np.array([d.memory_bytes for d in topo.devices], np.int64),
        bw=np.array(topo.bandwidth, np.float64),
    )


def instance_from_arrays(a) -> tuple[GroupedGraph, DeviceTopology]:
    types = [str(t) for t in a["types"]]
    sp = a["shape_ptr"]
    dims = a["shape_dims"]
    ops = [
        Operation(i, f"op{i}", types[int(a["op_type"][i])], float(a["op_cost"][i]),
                  tuple(int(x) for x in dims[sp[i]:sp[i + 1]]), int(a["op_param"][i]))
        for i in range(len(a["op_type"]))
    ]
    edges = [Edge(int(s), int(d), int(b))
             for s, d, b in zip(a["edge_src"], a["edge_dst"], a["edge_bytes"])]
    pp, po = a["part_ptr"], a["part_ops"]
    parts = [tuple(int(x) for x in po[pp[i]:pp[i + 1]]) for i in range(len(pp) - 1)]
    gg = GroupedGraph(ComputationGraph(ops, edges), parts)
    devs = [Device(i, "gpu" if int(k) else "cpu", float(r), int(m))
            for i, (k, r, m) in enumerate(zip(a["dev_kind"], a["dev_rate"], a["dev_mem"]))]
    topo = DeviceTopology(devs, [[float(x) for x in row] for row in a["bw"]])
    return gg, topo


def save_instance(path, gg, topo, **extra):
    np.savez_compressed(path, **instance_arrays(gg, topo), **extra)


def load_instance(path):
    with np.load(path, allow_pickle=False) as a:
        return instance_from_arrays(a)
