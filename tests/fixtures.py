"""Loaders for the committed golden fixtures (tests/golden/, made by make_golden.py)."""

from __future__ import annotations

import functools
import json
import os

import numpy as np

from paper_1706_04972_b200.instances import instance_from_arrays

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def npz(name):
    with np.load(os.path.join(GOLDEN, name), allow_pickle=False) as a:
        return {k: a[k] for k in a.files}


@functools.lru_cache(maxsize=None)
def cfg(name):
    """(GroupedGraph, DeviceTopology, K, raw arrays) for config C1/C2/C3/C3tight/C5."""
    a = npz(f"cfg_{name}.npz")
    gg, topo = instance_from_arrays(a)
    return gg, topo, int(a["K"]), a


def random_cases():
    """Unpack sim_random.npz into a list of (gg, topo, placement, expected dict)."""
    a = npz("sim_random.npz")
    keys = [k[:-5] for k in a if k.endswith("__ptr") and k[:-5] not in
            ("placement", "dev")]
    n = len(a["makespan"])
    cases = []
    for i in range(n):
        inst = {}
        for k in keys:
            ptr = a[k + "__ptr"]
            flat = a[k][ptr[i]:ptr[i + 1]]
            s1 = int(a[k + "__shape1"][i])
            inst[k] = flat.reshape(-1, s1) if s1 else flat
        inst["types"] = np.array(str(a["types_joined"][i]).split("|"))
        gg, topo = instance_from_arrays(inst)
        pp, dp = a["placement__ptr"], a["dev__ptr"]
        exp = dict(makespan=a["makespan"][i], busy=a["busy"][dp[i]:dp[i + 1]],
                   transfer=a["transfer"][dp[i]:dp[i + 1]], peak=a["peak"][dp[i]:dp[i + 1]],
                   feasible=bool(a["feasible"][i]), order=a["order"][pp[i]:pp[i + 1]],
                   oracle_sim=a["oracle_sim_makespan"][i])
        cases.append((gg, topo, [int(x) for x in a["placement"][pp[i]:pp[i + 1]]], exp))
    return cases


def train_golden(name):
    a = npz(f"train_{name}.npz")
    a["cfg"] = json.loads(str(a["cfg"]))
    a["csv"] = str(a["csv"])
    return a


def baseline_cases():
    """tests/golden/baselines.npz: [(gg, topo, bf_placement | None, bf_makespan, rs_budget, rs_placement | None)]
    from the reference's brute_force / place_random_search (make_golden.py baselines)."""
    a = npz("baselines.npz")
    out = []
    for i in range(int(a["n"])):
        pre = f"i{i}_"
        inst = {k[len(pre):]: v for k, v in a.items() if k.startswith(pre)}
        gg, topo = instance_from_arrays(inst)
        bf = [int(x) for x in inst["bf_placement"]] if inst["bf_placement"].size else None
        rs = [int(x) for x in inst["rs_placement"]] if inst["rs_placement"].size else None
        out.append((gg, topo, bf, float(inst["bf_makespan"]), int(inst["rs_budget"]), rs))
    return out, [int(x) for x in a["c1_rs_placement"]]


# Final parameters after Adam vs the reference / oracle: Adam's per-coordinate
# m / sqrt(v) carries rounding-level gradient differences (the decoder weight
# gradients are int8-digit tensor-core sums, ~1e-13 relative) into parameter
# differences of the same relative size on every coordinate; training logs
# stay byte-identical.  Gradients themselves are checked at 1e-9.
PARAM_RTOL = 1e-10
