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
