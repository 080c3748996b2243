"""Placement scorer: batched event-driven execution-time simulation on the GPU.

Drop-in for the reference cost model (``pkg/simulator.py``): same public names,
signatures, exceptions and return types.  Every scoring call runs the
``dp_simulate_batch`` sm_100a kernel (``csrc/sim.cu``) through the C-ABI in
``include/devplace_b200.h``; there is no CPU fallback.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

INFEASIBLE = math.inf


class TopologyError(ValueError):
    """Schema violation in a topology (reference ``pkg/simulator.py:41``)."""


@dataclass(frozen=True)
class Device:
    id: int
    kind: str
    compute_rate: float
    memory_bytes: int


class DeviceTopology:
    """Devices plus a dense directed bandwidth matrix (reference ``pkg/simulator.py:53-81``)."""

    def __init__(self, devices, bandwidth):
        self.devices = list(devices)
        self.bandwidth = [list(map(float, row)) for row in bandwidth]
        d = len(self.devices)
        for i, dev in enumerate(self.devices):
            if dev.id != i:
                raise TopologyError(f"device ids must be dense 0..{d - 1}; got {dev.id} at {i}")
            if dev.kind not in ("cpu", "gpu"):
                raise TopologyError(f"device {dev.id}: kind must be 'cpu' or 'gpu'")
            if not dev.compute_rate > 0:
                raise TopologyError(f"device {dev.id}: compute_rate must be > 0")
            if not dev.memory_bytes > 0:
                raise TopologyError(f"device {dev.id}: memory_bytes must be > 0")
        if len(self.bandwidth) != d or any(len(r) != d for r in self.bandwidth):
            raise TopologyError("bandwidth must be a DxD matrix")
        for i in range(d):
            for j in range(d):
                if i != j and not self.bandwidth[i][j] > 0:
                    raise TopologyError(f"bandwidth[{i}][{j}] must be > 0")

    @property
    def num_devices(self) -> int:
        return len(self.devices)

    def gpu_ids(self) -> list[int]:
        return [d.id for d in self.devices if d.kind == "gpu"]


@dataclass
class SimReport:
    makespan_seconds: float
    per_device_busy_seconds: list
    per_device_transfer_seconds: list
    per_device_peak_bytes: list
    feasible: bool


@dataclass(frozen=True)
class NoiseSpec:
    sigma: float
    seed: int = 0


def default_topology(num_gpus: int = 2, cpu_rate: float = 1.0, gpu_rate: float = 10.0,
                     cpu_gpu_bw: float = 16384.0, gpu_gpu_bw: float = 65536.0,
                     cpu_mem: int = 4 << 30, gpu_mem: int = 1 << 30) -> DeviceTopology:
    """One CPU then ``num_gpus`` GPUs (reference ``pkg/simulator.py:304-323``)."""
    devs = [Device(0, "cpu", cpu_rate, cpu_mem)]
    devs += [Device(1 + i, "gpu", gpu_rate, gpu_mem) for i in range(num_gpus)]
    n = len(devs)
    bw = [[0.0 if i == j else (gpu_gpu_bw if devs[i].kind == devs[j].kind == "gpu" else cpu_gpu_bw)
           for j in range(n)] for i in range(n)]
    return DeviceTopology(devs, bw)


# ----------------------------------------------------------------------------- device path
import threading as _threading  # noqa: E402
import weakref as _weakref  # noqa: E402

import numpy as _np  # noqa: E402


def graph_arrays(gg, topo) -> dict:
    """Host arrays by topological rank for dp_graph_create (include/devplace_b200.h).

    Mirrors the per-call setup of pkg/simulator.py:122-144 (rank, pending counts,
    out-edges by destination rank) and check_memory's resident bytes
    (pkg/simulator.py:101-102)."""
    n = gg.num_groups
    gid = _np.asarray(gg.topo, _np.int32).reshape(n)
    rank = _np.asarray(gg.topo_rank, _np.int64).reshape(n)
    cost = _np.array([gg.groups[g].compute_cost for g in gid], _np.float64).reshape(n)
    indeg = _np.array([len(gg.in_groups[g]) for g in gid], _np.int32).reshape(n)
    resident = _np.array([gg.groups[g].param_bytes + gg.groups[g].out_bytes for g in gid],
                         _np.int64).reshape(n)
    es = _np.array([(rank[e.src], rank[e.dst], e.tensor_bytes) for e in gg.group_edges],
                   _np.int64).reshape(-1, 3)
    es = es[_np.lexsort((es[:, 1], es[:, 0]))] if len(es) else es
    out_off = _np.zeros(n + 1, _np.int32)
    _np.add.at(out_off, es[:, 0] + 1, 1)
    out_off = _np.cumsum(out_off).astype(_np.int32)
    d = topo.num_devices
    return dict(
        n=n, d=d, cost=cost, indeg=indeg, out_off=out_off,
        out_dst=_np.ascontiguousarray(es[:, 1].astype(_np.int32)),
        out_bytes=_np.ascontiguousarray(es[:, 2].astype(_np.int64)),
        resident=resident, gid=gid,
        rate=_np.array([dv.compute_rate for dv in topo.devices], _np.float64),
        bw=_np.ascontiguousarray(_np.array(topo.bandwidth, _np.float64).reshape(d, d)),
        mem=_np.array([dv.memory_bytes for dv in topo.devices], _np.int64),
    )


def _hp(a):
    return a.ctypes.data if a.size else None


class DeviceGraph:
    """A grouped graph + topology resident on the current CUDA device (dp_graph)."""

    def __init__(self, gg, topo):
        import ctypes

        import torch

        from . import _native as nat

        self.n, self.d = gg.num_groups, topo.num_devices
        self.device = torch.device("cuda", torch.cuda.current_device())
        a = graph_arrays(gg, topo)
        self.arrays = a
        h = ctypes.c_void_p()
        rc = nat.lib().dp_graph_create(
            a["n"], a["d"], _hp(a["cost"]), _hp(a["indeg"]), _hp(a["out_off"]), _hp(a["out_dst"]),
            _hp(a["out_bytes"]), _hp(a["resident"]), _hp(a["gid"]), _hp(a["rate"]), _hp(a["bw"]),
            _hp(a["mem"]), ctypes.byref(h))
        nat.check(rc, "dp_graph_create")
        self.handle = h.value
        self._destroy = nat.lib().dp_graph_destroy
        self.gid_of_rank = torch.as_tensor(a["gid"].astype(_np.int64), device=self.device)

    def __del__(self):
        h = getattr(self, "handle", None)
        if h:
            try:
                self._destroy(h)
            except Exception:
                pass
            self.handle = None

    def simulate(self, placements, by_rank=False, order=False, stream=None, out=None):
        """Batched scorer: ``placements`` uint8 CUDA tensor [K, n].  Returns a dict
        of CUDA tensors (makespan, busy, transfer, peak, feasible[, order], err)."""
        import torch

        from . import _native as nat

        K = placements.shape[0]
        dev = placements.device
        if out is None:
            out = dict(
                makespan=torch.empty(K, dtype=torch.float64, device=dev),
                busy=torch.empty(K, self.d, dtype=torch.float64, device=dev),
                transfer=torch.empty(K, self.d, dtype=torch.float64, device=dev),
                peak=torch.empty(K, self.d, dtype=torch.int64, device=dev),
                feasible=torch.empty(K, dtype=torch.uint8, device=dev),
                err=torch.zeros(1, dtype=torch.uint8, device=dev),
            )
            if order:
                out["order"] = torch.empty(K, self.n, dtype=torch.int32, device=dev)
        rc = nat.lib().dp_simulate_batch(
            self.handle, K, nat.ptr(placements), 1 if by_rank else 0, nat.ptr(out["makespan"]),
            nat.ptr(out["busy"]), nat.ptr(out["transfer"]), nat.ptr(out["peak"]),
            nat.ptr(out["feasible"]), nat.ptr(out.get("order")), nat.ptr(out["err"]),
            nat.stream_ptr(stream))
        nat.check(rc, "dp_simulate_batch")
        return out


_cache_lock = _threading.Lock()
_cache: dict = {}


def device_graph(gg, topo) -> DeviceGraph:
    """Upload once per (graph, topology, CUDA device); later calls reuse the handle."""
    import torch

    key = (id(gg), id(topo), torch.cuda.current_device())
    with _cache_lock:
        ent = _cache.get(key)
        if ent is not None and ent[0]() is gg and ent[1]() is topo:
            return ent[2]
        dg = DeviceGraph(gg, topo)
        try:
            _cache[key] = (_weakref.ref(gg), _weakref.ref(topo), dg)
        except TypeError:  # objects without weakref support: no caching
            pass
        if len(_cache) > 64:
            for k in list(_cache)[:16]:
                _cache.pop(k, None)
        return dg


def _check_placement(gg, topo, placement):
    """Reference validation and messages (pkg/simulator.py:109-116)."""
    if len(placement) != gg.num_groups:
        raise ValueError(f"placement length {len(placement)} != group count {gg.num_groups}")
    for gid, dev in enumerate(placement):
        if not (0 <= dev < topo.num_devices):
            raise ValueError(f"group {gid}: device id {dev} out of range")


def _placements_tensor(placements, n, device):
    import torch

    if isinstance(placements, torch.Tensor):
        t = placements.to(device=device, dtype=torch.uint8)
    else:
        t = torch.as_tensor(_np.asarray(placements, _np.uint8).reshape(-1, n), device=device)
    return t.reshape(-1, n).contiguous()


def simulate_batch(gg, topo, placements, by_rank=False, order=False):
    """Score K placements at once on the GPU (K x n, by gid unless ``by_rank``)."""
    dg = device_graph(gg, topo)
    pl = _placements_tensor(placements, gg.num_groups, dg.device)
    out = dg.simulate(pl, by_rank=by_rank, order=order)
    return out


def simulate(gg, topo, placement) -> SimReport:
    """Drop-in for pkg/simulator.py:122-194 (runs the K-sim kernel with K=1)."""
    _check_placement(gg, topo, placement)
    out = simulate_batch(gg, topo, [list(placement)])
    mk = float(out["makespan"][0].item())
    return SimReport(
        makespan_seconds=mk,
        per_device_busy_seconds=out["busy"][0].tolist(),
        per_device_transfer_seconds=out["transfer"][0].tolist(),
        per_device_peak_bytes=[int(x) for x in out["peak"][0].tolist()],
        feasible=bool(out["feasible"][0].item()),
    )


def check_memory(gg, topo, placement):
    """Drop-in for pkg/simulator.py:93-106 (peaks computed by the same kernel)."""
    rep = simulate(gg, topo, placement)
    return rep.per_device_peak_bytes, rep.feasible


def measure(gg, topo, placement, noise: NoiseSpec | None = None, steps: int = 10) -> float:
    """Drop-in for pkg/simulator.py:205-223.  The simulator is pure, so the base
    makespan comes from one kernel evaluation; the optional lognormal noise
    factors are the reference's own numpy stream."""
    if steps < 2:
        raise ValueError("measure needs at least 2 steps (the first is discarded)")
    rep = simulate(gg, topo, placement)
    if not rep.feasible:
        return INFEASIBLE
    base = rep.makespan_seconds
    if noise is None:
        return base
    rng = _np.random.default_rng(noise.seed)
    factors = _np.exp(noise.sigma * rng.standard_normal(steps))
    return float(_np.mean(base * factors[1:]))
