"""K-sharded data parallelism for the REINFORCE step.

Samples are independent given the parameter snapshot and the simulator is
pure, so rank r of N owns samples [r*K/N, (r+1)*K/N): it replays exactly
those PCG64 draws (draw index = update*K*T + k*T + t — no RNG communication),
samples, scores and back-propagates them.  Two exchanges per update:

* all-gather of one small record per rank (``dp_exchange_pack``): the shard's
  makespans (f64) and feasibility (u8) plus the placement row of the shard's
  best candidate (first feasible sample with the smallest reward) — K*9 + N*T
  bytes instead of all K*T placements; every rank then replays the reference's
  sequential best / mean / baseline logic (pkg/trainer.py:281-304) on identical
  data (bit-identical state), and the global best row is the owning rank's
  candidate;
* sum all-reduce of the advantage-weighted fp64 gradient (P*8 = 532 KB) ->
  replicated Adam.

Transports (all expose ``all_gather(out, local)`` / ``all_reduce_sum(t)``):

* ``NcclExchange`` — NCCL over NVLink/NVSwitch through the library's own
  binding (csrc/comm.cu): one communicator per process (torchrun, ids
  broadcast over the torch.distributed group) or one per device in a single
  process (``ncclCommInitAll``).  Enqueued on the step's stream, so the whole
  update — collectives included — is captured in one CUDA graph.
* ``TorchExchange`` — torch.distributed (gloo, host-staged): CPU tests and
  several ranks sharing one GPU (``DP_DIST_BACKEND=gloo``).
* ``LocalGroup`` — in-process ranks on ONE device (the single-process
  multi-device runner's collectives when every "device" is the same GPU; used
  to test that orchestration on a one-GPU box).
"""

from __future__ import annotations

import ctypes


def shard(K: int, rank: int, size: int) -> tuple[int, int]:
    """(k_offset, K_local) of ``rank`` — contiguous, equal shards."""
    if size < 1 or not (0 <= rank < size):
        raise ValueError(f"bad rank {rank} of {size}")
    if K % size:
        raise ValueError(f"k={K} must be divisible by the number of ranks {size}")
    k_local = K // size
    return rank * k_local, k_local


def draw_index(update: int, k: int, t: int, K: int, T: int) -> int:
    """Index of the Generator.random() draw used by sample k, step t of an update
    (reference consumption order: K forward_sample calls of T draws each)."""
    return update * K * T + k * T + t


class TorchExchange:
    """The per-update collectives over a torch.distributed group."""

    capturable = False

    def __init__(self, group=None, backend: str | None = None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.backend = backend or dist.get_backend(group)
        self.size = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.capturable = self.backend == "nccl"

    def _host_staged(self, t):
        return self.backend != "nccl" and t.is_cuda

    def all_gather(self, out, local, stream=None):
        """out[N * len(local)] <- concatenation of every rank's local (rank order)."""
        if self.backend == "nccl":
            self.dist.all_gather_into_tensor(out, local.contiguous(), group=self.group)
        elif self._host_staged(local):
            o = out.cpu()
            self._gather_list(o, local.cpu().contiguous())
            out.copy_(o)
        else:
            self._gather_list(out, local.contiguous())
        return out

    def _gather_list(self, out, local):
        parts = list(out.chunk(self.size, dim=0))
        bufs = [p.clone() for p in parts]
        self.dist.all_gather(bufs, local, group=self.group)
        for p, b in zip(parts, bufs):
            p.copy_(b)

    def all_reduce_sum(self, t, stream=None):
        dist = self.dist
        if self._host_staged(t):
            h = t.cpu()
            dist.all_reduce(h, group=self.group)
            t.copy_(h)
        else:
            dist.all_reduce(t, group=self.group)
        return t

    def all_reduce_min(self, t, stream=None):
        h = t.cpu() if self._host_staged(t) else t
        self.dist.all_reduce(h, op=self.dist.ReduceOp.MIN, group=self.group)
        if h is not t:
            t.copy_(h)
        return t


# backwards-compatible name (round 1)
Exchange = TorchExchange


class _Comm:
    """Owner of one native dp_comm handle."""

    def __init__(self, handle, rank, size, device):
        from . import _native as nat

        self.handle, self.rank, self.size, self.device = handle, rank, size, device
        self._destroy = nat.lib().dp_comm_destroy

    def __del__(self):
        h = getattr(self, "handle", None)
        if h:
            try:
                self._destroy(h)
            except Exception:
                pass
            self.handle = None


def nccl_version() -> int:
    from . import _native as nat

    v = ctypes.c_int32()
    nat.check(nat.lib().dp_comm_version(ctypes.byref(v)), "dp_comm_version")
    return v.value


class NcclExchange:
    """NCCL collectives on the caller's stream (csrc/comm.cu; CUDA-graph capturable)."""

    capturable = True

    def __init__(self, comm: _Comm):
        self.comm, self.rank, self.size = comm, comm.rank, comm.size

    @classmethod
    def from_group(cls, group=None) -> "NcclExchange":
        """One communicator per process: rank 0 creates the NCCL id, the
        torch.distributed group broadcasts it (any backend)."""
        import torch
        import torch.distributed as dist

        from . import _native as nat

        rank, size = dist.get_rank(group), dist.get_world_size(group)
        buf = (ctypes.c_uint8 * 128)()
        if rank == 0:
            nat.check(nat.lib().dp_comm_unique_id(buf), "dp_comm_unique_id")
        obj = [bytes(buf) if rank == 0 else None]
        dist.broadcast_object_list(obj, src=dist.get_global_rank(group, 0) if group is not None else 0,
                                   group=group)
        uid = (ctypes.c_uint8 * 128).from_buffer_copy(obj[0])
        h = ctypes.c_void_p()
        nat.check(nat.lib().dp_comm_init_rank(size, uid, rank, ctypes.byref(h)), "dp_comm_init_rank")
        return cls(_Comm(h.value, rank, size, torch.cuda.current_device()))

    @staticmethod
    def init_all(devices) -> list:
        """One communicator per device, all in this process (ncclCommInitAll)."""
        from . import _native as nat

        n = len(devices)
        devs = (ctypes.c_int32 * n)(*devices)
        hs = (ctypes.c_void_p * n)()
        nat.check(nat.lib().dp_comm_init_all(n, devs, hs), "dp_comm_init_all")
        return [NcclExchange(_Comm(hs[i], i, n, devices[i])) for i in range(n)]

    def all_gather(self, out, local, stream=None):
        from . import _native as nat

        nbytes = local.numel() * local.element_size()
        if out.numel() * out.element_size() != nbytes * self.size:
            raise ValueError("all_gather: out must hold size x local bytes")
        nat.check(nat.lib().dp_comm_all_gather(self.comm.handle, nat.ptr(local), nat.ptr(out), nbytes,
                                               nat.stream_ptr(stream)), "dp_comm_all_gather")
        return out

    def all_reduce_sum(self, t, stream=None):
        from . import _native as nat

        nat.check(nat.lib().dp_comm_all_reduce_f64(self.comm.handle, nat.ptr(t), t.numel(), 0,
                                                   nat.stream_ptr(stream)), "dp_comm_all_reduce_f64")
        return t

    def all_reduce_min(self, t, stream=None):
        from . import _native as nat

        nat.check(nat.lib().dp_comm_all_reduce_f64(self.comm.handle, nat.ptr(t), t.numel(), 1,
                                                   nat.stream_ptr(stream)), "dp_comm_all_reduce_f64")
        return t


class nccl_group:
    """ncclGroupStart/End around per-device calls issued by one thread."""

    def __enter__(self):
        from . import _native as nat

        nat.check(nat.lib().dp_comm_group_start(), "dp_comm_group_start")
        return self

    def __exit__(self, *exc):
        from . import _native as nat

        nat.check(nat.lib().dp_comm_group_end(), "dp_comm_group_end")


class LocalGroup:
    """Collectives among in-process ranks that share one CUDA device and one
    stream: gathers are device copies, the sum runs in rank order."""

    capturable = True

    def __init__(self, size: int):
        self.size = size

    def all_gather(self, pairs):
        """pairs[r] = (out_r, local_r): every out_r <- concat(local_0..local_{N-1})."""
        for out, _ in pairs:
            n = pairs[0][1].numel()
            for r, (_, local) in enumerate(pairs):
                out.view(-1)[r * n:(r + 1) * n].copy_(local.view(-1))

    def all_reduce_sum(self, bufs):
        acc = bufs[0].clone()
        for b in bufs[1:]:
            acc += b
        for b in bufs:
            b.copy_(acc)

    def all_reduce_min(self, bufs):
        acc = bufs[0].clone()
        for b in bufs[1:]:
            acc = acc.minimum(b)
        for b in bufs:
            b.copy_(acc)


class NcclGroup:
    """The single-process multi-device collectives: one NcclExchange per device,
    every call wrapped in one NCCL group."""

    capturable = True

    def __init__(self, exchanges, streams):
        self.xs, self.streams = exchanges, streams
        self.size = len(exchanges)

    def all_gather(self, pairs):
        with nccl_group():
            for x, s, (out, local) in zip(self.xs, self.streams, pairs):
                x.all_gather(out, local, stream=s)

    def all_reduce_sum(self, bufs):
        with nccl_group():
            for x, s, b in zip(self.xs, self.streams, bufs):
                x.all_reduce_sum(b, stream=s)

    def all_reduce_min(self, bufs):
        with nccl_group():
            for x, s, b in zip(self.xs, self.streams, bufs):
                x.all_reduce_min(b, stream=s)
