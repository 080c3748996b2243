"""Search baselines as batched K-sim fan-outs.

Drop-in for the reference's exhaustive and random-search baselines
(``pkg/baselines.py:227-273``): same names, arguments, exceptions and
tie-breaking, with every candidate scored by the sm_100a simulator kernel in
batches instead of one ``simulate()`` call at a time.

* ``brute_force`` enumerates ``itertools.product(range(D), repeat=N)`` on
  the device (``dp_enumerate_placements``), scores each batch and folds the
  first strict minimum into a running best (``dp_argmin_feasible``), so ties
  resolve to the lexicographically smallest placement like the reference's
  sequential ``if makespan < best``.
* ``place_random_search`` draws candidates from the reference's own numpy
  stream on the host (``rng.integers(0, D, size=N)`` per candidate, duplicates
  skipped without consuming budget), then scores all distinct candidates on
  the device and returns the first best in draw order.

The heuristic baselines (single device, expert contiguous, min-cut) are
one-time host partitioners, not a K-sim fan-out, and stay out of scope
(DESIGN.md §8); ``place_single`` is kept because it is trivial.
"""

from __future__ import annotations

import numpy as np

from .simulator import device_graph


class NoFeasiblePlacement(RuntimeError):
    """No placement satisfying the memory model exists (or none was found)."""


class SearchSpaceTooLarge(RuntimeError):
    """Brute force would exceed its enumeration cap."""


_BATCH = 1 << 16


def place_single(gg, topo, device: int) -> list[int]:
    """Everything on one device (``pkg/baselines.py:30-34``)."""
    if not (0 <= device < topo.num_devices):
        raise ValueError(f"device id {device} out of range")
    return [device] * gg.num_groups


def _fold(dg, pl, base, best_val, best_idx, stream=None):
    from . import _native as nat

    out = dg.simulate(pl, by_rank=False)
    nat.check(nat.lib().dp_argmin_feasible(pl.shape[0], nat.ptr(out["makespan"]), nat.ptr(out["feasible"]),
                                           base, nat.ptr(best_val), nat.ptr(best_idx), nat.stream_ptr(stream)),
              "dp_argmin_feasible")


def brute_force(gg, topo, cap: int = 1 << 20) -> tuple[list[int], float]:
    """Exact argmin of the simulator over all feasible placements
    (``pkg/baselines.py:254-273``); lexicographically smallest on ties."""
    import torch

    from . import _native as nat

    n, d = gg.num_groups, topo.num_devices
    space = d ** n
    if space > cap:
        raise SearchSpaceTooLarge(f"{space} placements exceed the cap of {cap}")
    dg = device_graph(gg, topo)
    dev = dg.device
    best_val = torch.full((1,), np.inf, dtype=torch.float64, device=dev)
    best_idx = torch.full((1,), -1, dtype=torch.int64, device=dev)
    buf = torch.empty(min(space, _BATCH), max(n, 1), dtype=torch.uint8, device=dev)
    for start in range(0, space, _BATCH):
        cnt = min(_BATCH, space - start)
        pl = buf[:cnt, :n]
        if n:
            nat.check(nat.lib().dp_enumerate_placements(n, d, start, cnt, nat.ptr(pl), None),
                      "dp_enumerate_placements")
        _fold(dg, pl, start, best_val, best_idx)
    idx = int(best_idx.item())
    if idx < 0:
        raise NoFeasiblePlacement("every placement violates device memory")
    digits, c = [0] * n, idx
    for g in range(n - 1, -1, -1):
        digits[g], c = c % d, c // d
    return digits, float(best_val.item())


def place_random_search(gg, topo, budget: int, seed: int = 0) -> list[int] | None:
    """Best feasible of ``budget`` distinct uniform placements, None if none
    (``pkg/baselines.py:227-251``)."""
    import torch

    from . import _native as nat

    if budget < 1:
        raise ValueError("budget must be >= 1")
    n, d = gg.num_groups, topo.num_devices
    rng = np.random.default_rng(seed)
    total = d ** n
    seen, cands = set(), []
    while len(seen) < min(budget, total):
        candidate = tuple(int(x) for x in rng.integers(0, d, size=n))
        if candidate in seen:
            continue
        seen.add(candidate)
        cands.append(candidate)
    dg = device_graph(gg, topo)
    dev = dg.device
    best_val = torch.full((1,), np.inf, dtype=torch.float64, device=dev)
    best_idx = torch.full((1,), -1, dtype=torch.int64, device=dev)
    arr = np.asarray(cands, np.uint8).reshape(len(cands), n)
    for start in range(0, len(cands), _BATCH):
        pl = torch.as_tensor(arr[start:start + _BATCH], device=dev).contiguous()
        _fold(dg, pl, start, best_val, best_idx)
    idx = int(best_idx.item())
    return None if idx < 0 else list(cands[idx])
