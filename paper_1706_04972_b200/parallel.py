"""K-sharded data parallelism for the REINFORCE step.

Samples are independent given the parameter snapshot and the simulator is
pure, so rank r of N owns samples [r*K/N, (r+1)*K/N): it replays exactly
those PCG64 draws (draw index = update*K*T + k*T + t — no RNG communication),
samples, scores and back-propagates them.  One exchange per update:

* all-gather of the per-sample scores (makespan f64, feasible u8) and
  placements (u8 by rank) -> every rank replays the reference's sequential
  best / mean / baseline logic on identical data (bit-identical state);
* all-reduce (sum) of the advantage-weighted gradient -> replicated Adam.

Collectives go through torch.distributed: NCCL over NVLink on B200 (the
production path, CUDA-graph capturable), gloo for CPU tests and for
exercising the multi-rank code path with several ranks on one GPU
(``DP_DIST_BACKEND=gloo``, host-staged).
"""

from __future__ import annotations


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


class Exchange:
    """The per-update collectives of a K-sharded controller."""

    def __init__(self, group=None, backend: str | None = None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.backend = backend or dist.get_backend(group)
        self.size = dist.get_world_size(group)

    def _host_staged(self, t):
        return self.backend != "nccl" and t.is_cuda

    def all_gather(self, out, local):
        """out[K, ...] <- concatenation of every rank's local[K/N, ...] (rank order)."""
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

    def all_reduce_sum(self, t):
        dist = self.dist
        if self._host_staged(t):
            h = t.cpu()
            dist.all_reduce(h, group=self.group)
            t.copy_(h)
        else:
            dist.all_reduce(t, group=self.group)
        return t
