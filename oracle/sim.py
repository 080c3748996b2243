"""TEST INFRASTRUCTURE ONLY — ctypes front-end of the C simulator restatement.

Reference: /root/reference/pkg/src/devplace/simulator.py:93-194 (see sim_oracle.c).
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = os.path.join(_HERE, "liboracle_sim.so")
_lib = None


def build():
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(
                os.path.join(_HERE, "sim_oracle.c")):
            build()
        L = ctypes.CDLL(_LIB)
        P = ctypes.c_void_p
        L.oracle_simulate_batch.argtypes = [ctypes.c_int, P, P, P, P, P, P, P, ctypes.c_int, P, P, P,
                                            ctypes.c_int, P, P, P, P, P, P, P, ctypes.c_int, P]
        L.oracle_simulate_batch.restype = ctypes.c_int
        _lib = L
    return _lib


class OracleGraph:
    """Graph + topology arrays by gid (reference GroupedGraph fields, pkg/graph.py:183-238)."""

    def __init__(self, gg, topo):
        n = gg.num_groups
        rank = np.asarray(gg.topo_rank, np.int32)
        self.n, self.d = n, topo.num_devices
        self.cost = np.array([g.compute_cost for g in gg.groups], np.float64)
        self.rank = rank
        self.indeg = np.array([len(gg.in_groups[i]) for i in range(n)], np.int32)
        rows = [[] for _ in range(n)]
        for e in gg.group_edges:
            rows[e.src].append((int(rank[e.dst]), e.dst, e.tensor_bytes))
        self.eoff = np.zeros(n + 1, np.int32)
        dst, byt = [], []
        for i, r in enumerate(rows):
            r.sort()  # simulator.py:143, ascending destination rank
            dst.extend(x[1] for x in r)
            byt.extend(x[2] for x in r)
            self.eoff[i + 1] = len(dst)
        self.edst = np.array(dst, np.int32)
        self.ebytes = np.array(byt, np.int64)
        self.resident = np.array([g.param_bytes + g.out_bytes for g in gg.groups], np.int64)
        self.rate = np.array([dv.compute_rate for dv in topo.devices], np.float64)
        self.bw = np.array(topo.bandwidth, np.float64).reshape(-1)
        self.mem = np.array([dv.memory_bytes for dv in topo.devices], np.int64)

    def simulate(self, placements, order=False, threads=1):
        pl = np.ascontiguousarray(np.asarray(placements, np.int64).reshape(-1, self.n))
        if pl.size and (pl.min() < 0 or pl.max() >= self.d):
            raise ValueError("device id out of range")
        pl = pl.astype(np.uint8)
        K, d = pl.shape[0], self.d
        out = dict(makespan=np.zeros(K), busy=np.zeros((K, d)), transfer=np.zeros((K, d)),
                   peak=np.zeros((K, d), np.int64), feasible=np.zeros(K, np.uint8))
        ordr = np.zeros((K, self.n), np.int32) if order else None
        bad = ctypes.c_int(-1)
        p = lambda a: a.ctypes.data if a is not None and a.size else None  # noqa: E731
        rc = lib().oracle_simulate_batch(
            self.n, p(self.cost), p(self.rank), p(self.indeg), p(self.eoff), p(self.edst),
            p(self.ebytes), p(self.resident), d, p(self.rate), p(self.bw), p(self.mem), K, p(pl),
            p(out["makespan"]), p(out["busy"]), p(out["transfer"]), p(out["peak"]),
            p(out["feasible"]), p(ordr), threads, ctypes.byref(bad))
        if rc:
            raise ValueError(f"placement {bad.value}: device id out of range")
        if order:
            out["order"] = ordr
        return out
