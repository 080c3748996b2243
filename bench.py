#!/usr/bin/env python
"""Benchmark: batched REINFORCE placement step on B200 (BASELINE.json metric).

One "step" = one full REINFORCE update of the device-placement policy on the
Inception-V3-shaped graph (config C3: 256 co-location groups, 4 simulated GPUs,
K=256 samples per B200): encoder, K sampled placements (PCG64 replay of the
reference's RNG stream), K event-exact simulations, rewards/baseline,
policy-gradient backward, [NCCL all-reduce], Adam.  Nothing is skipped; the
precision is the reference's (fp64).

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]
    torchrun --nproc-per-node N bench.py --gpus N ...   (K per GPU fixed: weak scaling)

Prints ONE JSON line (rank 0).  See DESIGN.md §6 for the roofline terms.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "placements sampled+scored/sec"
UNIT = "placements/s"
CFG_FILE = {"C1": "cfg_C1.npz", "C2": "cfg_C2.npz", "C3": "cfg_C3.npz", "C3tight": "cfg_C3tight.npz",
            "C5": "cfg_C5.npz"}
CFG_DESC = {
    "C1": "rnnlm_grid L2 S16 -> 100 co-location groups, 252 group edges, cpu+1gpu",
    "C2": "nmt_attention L4 S11 -> 243 co-location groups, 853 group edges, cpu+4gpu",
    "C3": "inception_blocks B18 br4 -> 256 co-location groups, 454 group edges, 4 simulated GPUs "
          "(rate 10, 65536 B/s links)",
    "C3tight": "C3 graph, 30 MiB per simulated GPU (memory-tight)",
    "C5": "random DAG 20k ops -> 2000 groups, 5969 group edges, cpu+7gpu",
    "C4": "mixed batch: C1 (rnnlm, 100 groups, cpu+1gpu) + C2 (nmt, 243 groups, cpu+4gpu) as two independent "
          "tasks (own parameters, stores, RNG), K=512 each per GPU, one CUDA-graph replay per round",
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None,
                    help="timed steps (default: enough for a >= ~0.4 s timed region, so the 100 ms "
                         "nvidia-smi clock sampler sees it; 20 for the reference arm and the long configs)")
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="C3")
    ap.add_argument("--k-per-gpu", type=int, default=None)
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--cpu-sample", type=int, default=None, help="placements in the CPU baseline sample")
    ap.add_argument("--skip-cpu", action="store_true")
    ap.add_argument("--profile-phases", type=int, default=3)
    ap.add_argument("--mode", choices=["step", "sim"], default="step",
                    help="step: full REINFORCE update (headline); sim: scorer only (placements scored/s)")
    ap.add_argument("--sim-k", type=int, default=65536, help="placements per scorer-only step")
    ap.add_argument("--single-process", action="store_true",
                    help="one process drives --gpus N devices (MultiDeviceRunner, NCCL ncclCommInitAll); "
                         "with fewer visible GPUs the ranks share cuda:0")
    args = ap.parse_args()
    if args.steps is None:
        if args.impl == "reference" or args.config == "C5":
            args.steps = 20
        elif args.mode == "sim":
            args.steps = 60
        else:
            args.steps = 100 if args.config == "C4" else 200
    return args


def load_config(name):
    from paper_1706_04972_b200.instances import load_instance
    import numpy as np

    path = os.path.join(ROOT, "tests", "golden", CFG_FILE[name])
    gg, topo = load_instance(path)
    with np.load(path) as a:
        K = int(a["K"])
    return gg, topo, K


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi sampling DURING the timed region (B200_PROFILING.md clocks line)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index, self.rows, self.proc, self.t_start, self.t_end = index, [], None, 0.0, None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                          "-i", str(self.index), "-lms", "100"], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
            # nvidia-smi takes a few hundred ms to start: wait for its first line
            # (taken before the region, dropped) so the region is sampled throughout
            t0 = time.monotonic()
            while not self.rows and time.monotonic() - t0 < 3.0:
                time.sleep(0.01)
        except FileNotFoundError:
            self.proc = None
        self.t_start = time.monotonic()
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append((time.monotonic(), [c.strip() for c in line.split(",")]))

    def __exit__(self, *exc):
        self.t_end = time.monotonic()
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        # only samples taken inside the timed region (a line is read a few ms after
        # nvidia-smi takes it); if the region was shorter than the sampling period,
        # the first sample after it, flagged
        inside = [r for t, r in self.rows if t > self.t_start and (self.t_end is None or t <= self.t_end + 0.02)]
        note = None
        if not inside and self.rows:
            after = [r for t, r in self.rows if t > self.t_start] or [self.rows[-1][1]]
            inside, note = after[:1], "timed region shorter than the 100 ms sampling period: first sample after it"
        if not inside:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[1]) for r in inside if len(r) > 2 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in inside if len(r) > 2 and r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in inside:
            for i, nm in enumerate(names):
                if len(r) > 5 + i and r[5 + i].lower() == "active":
                    reasons.add(nm)
        out = {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
               "reasons": sorted(reasons), "samples": len(inside)}
        if note:
            out["note"] = note
        return out


# ----------------------------------------------------------------------------- roofline terms
def decoder_flops_per_placement(T, D, dd=16, H=64):
    """Algorithmic FLOPs of one sampled placement in the reference's decoder
    (pkg/policy.py:291-306): per step the gate contraction
    [x; h] @ W_dec 2*(dd+H)*4H, scores proj @ h 2*T*H, context alpha @ enc
    2*T*H, u = hc @ W_out 2*2H*dd, logits 2*dd*D.  (The kernel does less: the
    x half is a (D+1)-row table lookup and the context is folded into uc.)"""
    return T * (2 * (dd + H) * 4 * H + 4 * T * H + 2 * 2 * H * dd + 2 * dd * D)


def ncu_traffic(kernel, suffix=""):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of ``kernel`` from
    the latest committed ncu --set full capture of the workload (C3 K=256:
    profiles/rNN_ncu_summary.json; C5 K=4096: profiles/rNN_C5_ncu_summary.json)."""
    import glob

    files = sorted(glob.glob(os.path.join(ROOT, "profiles", f"r[0-9][0-9]{suffix}_ncu_summary.json")))
    for f in reversed(files):
        try:
            d = json.load(open(f)).get(kernel)
        except Exception:
            continue
        if d and "dram_bytes_per_launch" in d:
            return {"bytes_per_launch": d["dram_bytes_per_launch"], "source": os.path.relpath(f, ROOT)}
    return None


def policy_flops_per_placement(T, D, K):
    """BASELINE.md §5 F_pol (forward + backward GEMM flops per placement)."""
    return 3 * T * (45056 + 32 * D) + 768 * T * T + 258048 * T / K


def fp64_peak_tflops(nat, torch):
    scratch = torch.zeros(1, dtype=torch.float64, device="cuda")
    blocks, threads, iters = 148 * 8, 256, 4096
    best = 0.0
    for _ in range(4):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        nat.check(nat.lib().dp_fp64_fma_probe(blocks, threads, iters, scratch.data_ptr(),
                                              torch.cuda.current_stream().cuda_stream), "probe")
        e.record()
        torch.cuda.synchronize()
        ms = s.elapsed_time(e)
        best = max(best, blocks * threads * iters * 16 / (ms * 1e-3) / 1e12)
    return best


# ----------------------------------------------------------------------------- CPU baseline
def cfg_path(name):
    return os.path.join(ROOT, "tests", "golden", CFG_FILE[name])


def cpu_k_for(name, K):
    """Placements per timed CPU step: the config's own K where a reference update
    takes seconds on the host cores (C1-C4), a bounded sample for C5 (one
    reference placement there costs ~3 s of CPU)."""
    return K if name != "C5" else 2 * len(os.sched_getaffinity(0))


def cpu_baseline(names, ks):
    """The reference's own code (oracle/_ref, installed unmodified by
    oracle/make_ref.sh) on all host cores: one warm-up + one timed REINFORCE
    update per task (oracle/refarm.py).  Falls back to the oracle port when the
    reference install is absent."""
    sys.path.insert(0, ROOT)
    from oracle import refarm

    workers = len(os.sched_getaffinity(0))
    if not refarm.available():
        return cpu_baseline_port(names, ks)
    tot_p, tot_s, parts = 0, 0.0, []
    for name, K in zip(names, ks):
        k = cpu_k_for(name, K)
        r = refarm.time_steps(cfg_path(name), k, steps=1, warmup=1, workers=workers)
        tot_p += r["placements"]
        tot_s += r["seconds"]
        parts.append(f"{name}: one update of K={k} ({r['seconds']:.2f} s)")
    return {"value": tot_p / tot_s, "unit": UNIT, "cores": workers, "kind": "reference",
            "sample": "; ".join(parts) + " — the unmodified reference (oracle/_ref) forward_sample + measure + "
                      "grad_log_prob per placement on a persistent fork pool (BLAS 1 thread/process), reference "
                      "baseline/Adam in the parent, after one warm-up update"}


def cpu_baseline_port(names, ks):
    from oracle.trainer import cpu_step_rate

    workers = len(os.sched_getaffinity(0))
    tot_p, tot_s = 0, 0.0
    for name in names:
        gg, topo, _ = load_config(name)
        r = cpu_step_rate(gg, topo, 2 * workers, workers=workers)
        tot_p += r["placements"]
        tot_s += r["seconds"]
    return {"value": tot_p / tot_s, "unit": UNIT, "cores": workers, "kind": "port",
            "sample": f"{tot_p} placements (oracle port: numpy fp64 + C simulator restatement)"}


def reference_extras(name):
    """R1 (reference train() as shipped, one process) and R2 (reference simulate
    on all cores) for the reference line."""
    from oracle import refarm

    out = {}
    try:
        r1 = refarm.single_process_rate(cfg_path(name), k=16)
        out["r1_single_process"] = {"value": r1["rate"], "unit": UNIT, "cores": 1,
                                    "sample": f"reference train(k=16, 2 updates) in one process, "
                                              f"update 1 wall {r1['update_ms']:.0f} ms"}
    except Exception as ex:  # pragma: no cover
        out["r1_single_process"] = {"error": repr(ex)}
    try:
        n = 4096 if name != "C5" else 512
        r2 = refarm.scorer_rate(cfg_path(name), n=n)
        out["r2_scorer_only"] = {"value": r2["rate"], "unit": "placements scored/s", "cores": r2["workers"],
                                 "sample": f"reference simulate over {n} random placements, fork pool"}
    except Exception as ex:  # pragma: no cover
        out["r2_scorer_only"] = {"error": repr(ex)}
    return out


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    sys.path.insert(0, ROOT)
    from oracle import refarm

    workers = len(os.sched_getaffinity(0))
    if args.mode == "sim":
        name = args.config
        vals = []
        for _ in range(max(1, args.steps)):
            vals.append(refarm.scorer_rate(cfg_path(name), n=4096 if name != "C5" else 512)["rate"])
        value = statistics.median(vals)
        line = {"impl": "reference", "metric": "placements scored/sec (simulator only)", "value": value,
                "unit": "placements/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic", "config": {"workload": f"{name}: {CFG_DESC[name]}",
                                                "parallelism": f"cpu fork pool x{workers}"},
                "cpu_baseline": {"value": value, "unit": "placements/s", "cores": workers, "kind": "reference",
                                 "sample": "reference simulate over 4096 random placements per step"},
                "e2e": {"value": value, "unit": "placements/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return
    names = ["C1", "C2"] if args.config == "C4" else [args.config]
    ks = []
    for name in names:
        _, _, Kc = load_config(name)
        ks.append(512 if args.config == "C4" else Kc)
    kind = "reference" if refarm.available() else "port"
    tot_p, tot_s = 0, 0.0
    if kind == "reference":
        steppers = [refarm.RefStepper(cfg_path(n), cpu_k_for(n, k), workers=workers) for n, k in zip(names, ks)]
        try:
            for _ in range(max(0, args.warmup)):
                for st in steppers:
                    st.step()
            t0 = time.perf_counter()
            for _ in range(args.steps):
                for st in steppers:
                    tot_p += st.step()[0]
            tot_s = time.perf_counter() - t0
        finally:
            for st in steppers:
                st.close()
        sample = (f"{args.steps} timed updates (+{args.warmup} warm-up) of " +
                  " + ".join(f"{n} K={cpu_k_for(n, k)}" for n, k in zip(names, ks)) +
                  ": the unmodified reference (oracle/_ref) per placement on a persistent fork pool "
                  "(BLAS pinned to 1 thread), reference baseline + Adam in the parent")
    else:
        from oracle.trainer import cpu_step_rate

        for name in names:
            gg, topo, _ = load_config(name)
            for _ in range(args.steps):
                r = cpu_step_rate(gg, topo, 2 * workers, workers=workers)
                tot_p += r["placements"]
                tot_s += r["seconds"]
        sample = f"{args.steps} steps x {2 * workers} placements, oracle port (reference not installed)"
    value = tot_p / tot_s
    k_cpu = [cpu_k_for(n, k) for n, k in zip(names, ks)]
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": tot_s / args.steps * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": {"workload": f"{args.config}: {CFG_DESC[args.config]}",
                                    "k_per_step": k_cpu, "same_k_as_gpu_arm": k_cpu == ks,
                                    "parallelism": f"cpu fork pool x{workers}"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": workers, "kind": kind, "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    if kind == "reference":
        line.update(reference_extras(names[0]))
        r1 = line.get("r1_single_process", {}).get("value")
        if r1:
            line["per_core_vs_single_process"] = value / workers / r1
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- scorer-only arm
def sim_bytes_per_placement(n, e, d):
    """B_sim: algorithmic bytes per scored
    placement = 32N + 12E + 24D + 9."""
    return 32 * n + 12 * e + 24 * d + 9


def run_sim(args):
    """Placements scored/s through dp_simulate_batch (the K-sim kernel alone):
    ``--sim-k`` random placements (by group id) per GPU per step, resident in
    HBM; e2e adds the placements' H2D copy and the makespan/feasible D2H."""
    import numpy as np
    import torch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0")) % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_1706_04972_b200 import _native as nat
    from paper_1706_04972_b200 import simulator as S

    name = args.config if args.config in CFG_FILE else "C3"
    gg, topo, _ = load_config(name)
    n, d, K = gg.num_groups, topo.num_devices, args.sim_k
    dg = S.device_graph(gg, topo)
    host = np.random.default_rng(1 + rank).integers(0, d, (K, n)).astype(np.uint8)
    pl = torch.as_tensor(host, device="cuda")
    out = dg.simulate(pl)
    stream = torch.cuda.current_stream()
    l0 = nat.lib().dp_launch_count()
    for _ in range(max(1, args.warmup)):
        dg.simulate(pl, out=out)
    torch.cuda.synchronize()
    launches = (nat.lib().dp_launch_count() - l0) // max(1, args.warmup)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for i in range(args.steps):
            flush.fill_(float(i))
            evs[i][0].record(stream)
            dg.simulate(pl, out=out)
            evs[i][1].record(stream)
        torch.cuda.synchronize()
    ms = [a.elapsed_time(b) for a, b in evs]
    tot = sum(ms)
    # e2e: pinned host placements -> device, score, makespan + feasible -> host
    hpl = torch.from_numpy(host).pin_memory()
    hmk = torch.empty(K, dtype=torch.float64, pin_memory=True)
    hfe = torch.empty(K, dtype=torch.uint8, pin_memory=True)
    dpl = torch.empty_like(pl)
    e2e = []
    for i in range(args.steps):
        flush.fill_(1.0)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        dpl.copy_(hpl, non_blocking=True)
        o = dg.simulate(dpl, out=out)
        hmk.copy_(o["makespan"], non_blocking=True)
        hfe.copy_(o["feasible"], non_blocking=True)
        b.record(stream)
        torch.cuda.synchronize()
        e2e.append(a.elapsed_time(b))
    e2e_tot = sum(e2e)
    if world > 1:
        t = torch.tensor([tot, e2e_tot], dtype=torch.float64, device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        tot, e2e_tot = t.tolist()
    if rank != 0:
        torch.distributed.destroy_process_group()
        return
    value = K * world * args.steps / (tot * 1e-3)
    e = len(gg.group_edges)
    bsim = sim_bytes_per_placement(n, e, d)
    pk = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    peak = pk.get("hbm_gbs") or 7672.0
    per_launch_ms = tot / args.steps
    achieved = bsim * K / (per_launch_ms * 1e-3) / 1e9
    tr = ncu_traffic("sim_warp_kernel", "_sim") if (name, K) == ("C3", 65536) else None
    cpu = None
    if world == 1 and not args.skip_cpu:
        sys.path.insert(0, ROOT)
        from oracle import refarm

        if refarm.available():
            r2 = refarm.scorer_rate(cfg_path(name), n=4096 if name != "C5" else 512)
            cpu = {"value": r2["rate"], "unit": "placements/s", "cores": r2["workers"], "kind": "reference",
                   "sample": f"R2: reference simulate over {r2['placements']} random placements on a fork pool "
                             f"({r2['seconds']:.2f} s)"}
            # the kernel's makespans for the same placements equal the reference's
            chk = torch.as_tensor(np.random.default_rng(1).integers(0, d, (r2["placements"], n)).astype(np.uint8),
                                  device="cuda")
            mine = dg.simulate(chk)["makespan"].cpu().numpy()
            cpu["bit_exact_makespans"] = bool(np.array_equal(mine, r2["makespans"]))
    line = {
        "metric": "placements scored/sec (simulator only)", "value": value, "unit": "placements/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": tot / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{name}: {CFG_DESC[name]}", "k_per_gpu": K, "global_k": K * world,
                   "placements": "numpy default_rng(1 + rank) uniform device ids, by group id",
                   "parallelism": f"dp{world} (placements sharded, no collective)",
                   "l2": "flushed between timed steps (256 MiB write)"},
        "e2e": {"value": K * world * args.steps / (e2e_tot * 1e-3), "unit": "placements/s",
                "h2d_bytes_per_step": K * n, "d2h_bytes_per_step": K * 9,
                "note": "placements H2D from pinned host -> score -> makespan + feasible D2H"},
        "gpu_launches": launches * args.steps, "gpu_launches_per_step": launches,
        "roofline": {"kernel": "sim_warp_kernel (dp_simulate_batch)", "bound": "hbm", "achieved": achieved,
                     "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": (tr or {}).get("bytes_per_launch"),
                     "traffic_source": (tr or {}).get("source"),
                     "algorithmic_bytes_per_placement": bsim, "avg_launch_ms": per_launch_ms,
                     "peak_source": "MEASURED_PEAKS.json hbm_gbs" if pk.get("hbm_gbs") else "B200_PROFILING fallback"},
        "cpu_baseline": cpu, "clocks": clk.summary(),
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


# ----------------------------------------------------------------------------- single-process multi-GPU
def run_single_process(args):
    """``--single-process --gpus N``: one process, N GPUs, the plain train()
    path (trainer.MultiDeviceRunner): K = k_per_gpu * N sharded over the
    devices, NCCL between them, one CUDA graph per device replayed per update.
    Per-step time = max over devices of the CUDA-event interval on each
    device's stream (all devices synchronised on both sides)."""
    import numpy as np
    import torch

    import paper_1706_04972_b200 as dp
    from paper_1706_04972_b200 import _native as nat

    N = args.gpus
    vis = torch.cuda.device_count()
    devices = list(range(N)) if vis >= N else [0] * N
    name = args.config if args.config in CFG_FILE else "C3"
    gg, topo, K_cfg = load_config(name)
    k_gpu = args.k_per_gpu or K_cfg
    total_updates = args.warmup + 2 * args.steps + 4
    cfg = dp.TrainerConfig(k=k_gpu * N, total_updates=total_updates, seed=0, devices=tuple(devices))
    task = dp.trainer._make_task(gg, topo, cfg)
    seq = np.random.SeedSequence(cfg.seed).spawn(1)[0]
    runner = dp.trainer.MultiDeviceRunner(task, cfg, devices, seq)
    l0 = nat.lib().dp_launch_count()
    runner.step()
    for d in sorted(set(devices)):
        torch.cuda.synchronize(d)
    launches = nat.lib().dp_launch_count() - l0
    runner.capture()
    for _ in range(max(0, args.warmup - 1)):
        runner.replay()
    uniq = sorted(set(devices))
    flush = {d: torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=f"cuda:{d}") for d in uniq}
    streams = {d: s for d, s in zip(devices, runner.streams)}
    evs = [{d: (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for d in uniq}
           for _ in range(args.steps)]
    for d in uniq:
        torch.cuda.synchronize(d)
    with ClockSampler(uniq[0]) as clk:
        for i in range(args.steps):
            for d in uniq:
                with torch.cuda.device(d):
                    flush[d].fill_(float(i))
                    streams[d].wait_stream(torch.cuda.current_stream(d))
                    evs[i][d][0].record(streams[d])
            for g, d, s in runner._graphs:
                with torch.cuda.device(d), torch.cuda.stream(s):
                    g.replay()
            for d in uniq:
                with torch.cuda.device(d):
                    evs[i][d][1].record(streams[d])
                    torch.cuda.current_stream(d).wait_stream(streams[d])
        for d in uniq:
            torch.cuda.synchronize(d)
    step_ms = [max(evs[i][d][0].elapsed_time(evs[i][d][1]) for d in uniq) for i in range(args.steps)]
    tot = sum(step_ms)
    for c in runner.ctls:
        c.check_errors()
    K = cfg.k
    value = K * args.steps / (tot * 1e-3)
    # e2e: parameters from pinned host to every device's store, one update,
    # parameters + log row of rank 0 back
    hp = torch.empty(runner.stores[0].params.numel(), dtype=torch.float64, pin_memory=True)
    hp.copy_(runner.stores[0].params.cpu())
    ho = torch.empty_like(hp, pin_memory=True)
    hl = torch.empty(8, dtype=torch.float64, pin_memory=True)
    e2e = []
    for i in range(args.steps):
        t0 = time.perf_counter()
        for st, d in zip(runner.stores, devices):
            with torch.cuda.device(d):
                st.params.copy_(hp, non_blocking=True)
        runner.replay()
        with torch.cuda.device(devices[0]):
            ho.copy_(runner.stores[0].params, non_blocking=True)
            hl.copy_(runner.ctls[0].log[:8], non_blocking=True)
        for d in uniq:
            torch.cuda.synchronize(d)
        e2e.append((time.perf_counter() - t0) * 1e3)
        hp.copy_(ho)
    cert = runner.result([0.0] * runner.ctls[0].updates_done).sampling
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": N, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": tot / args.steps, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{name}: {CFG_DESC[name]}", "k_per_gpu": k_gpu, "global_k": K,
                   "parallelism": f"dp{N} single process (devices {devices}; "
                                  f"{'shared GPU, LocalGroup' if runner.shared_gpu else 'NCCL ncclCommInitAll'})",
                   "l2": "flushed between timed steps (256 MiB write)", "cuda_graph": True},
        "steps_per_sec": 1e3 / (tot / args.steps),
        "e2e": {"value": K * args.steps / (sum(e2e) * 1e-3), "unit": UNIT,
                "h2d_bytes_per_step": hp.numel() * 8 * len(devices), "d2h_bytes_per_step": hp.numel() * 8 + 64,
                "note": "host wall clock around params H2D (every device) -> graph replay -> params + log D2H"},
        "gpu_launches": launches * args.steps, "gpu_launches_per_step": launches,
        "sampling": cert, "clocks": clk.summary(),
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- our arm
def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    if args.mode == "sim":
        return run_sim(args)
    if args.single_process:
        return run_single_process(args)

    import numpy as np
    import torch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # DP_DIST_BACKEND=gloo exercises the multi-rank path with several ranks per GPU
    backend = os.environ.get("DP_DIST_BACKEND", "nccl")
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    group = None
    if world > 1:
        import torch.distributed as dist

        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
        group = dist.group.WORLD

    import paper_1706_04972_b200 as dp
    from paper_1706_04972_b200 import _native as nat

    # measurement A/B only: DP_DECODER_VARIANT=4 runs the opt-in tensor-core-gate decoder
    if os.environ.get("DP_DECODER_VARIANT"):
        nat.check(nat.lib().dp_debug_decoder_variant(int(os.environ["DP_DECODER_VARIANT"])), "variant")
    if os.environ.get("DP_ENCODER_VARIANT"):
        nat.check(nat.lib().dp_debug_encoder_variant(int(os.environ["DP_ENCODER_VARIANT"])), "variant")

    # C4 = the mixed batch: the C1 and C2 tasks (own parameters, stores, RNG
    # streams) advanced together, K=512 each
    names = ["C1", "C2"] if args.config == "C4" else [args.config]
    total_updates = args.warmup + 2 * args.steps + args.profile_phases + 8
    ctls, stores, K = [], [], 0
    for name in names:
        gg, topo, K_cfg = load_config(name)
        k_gpu = args.k_per_gpu or (512 if args.config == "C4" else K_cfg)
        cfg = dp.TrainerConfig(k=k_gpu * world, total_updates=total_updates, seed=0)
        task = dp.trainer._make_task(gg, topo, cfg)
        store = dp.ParameterStore(task.template.to_flat(), max_steps=total_updates + 1)
        seq = np.random.SeedSequence(cfg.seed).spawn(1)[0]
        ctls.append(dp.trainer.DeviceController(task, store, seq, 0, world=(rank, world, group)))
        stores.append(store)
        K += cfg.k
    ctl, store = ctls[0], stores[0]
    # several tasks: one stream each (one graph replay per round); under
    # torch.distributed they run back to back so every rank issues the same
    # collective order
    runner = ctl if len(ctls) == 1 else dp.trainer.ConcurrentRunner(ctls, concurrent=world == 1)
    stream = torch.cuda.current_stream()
    T = ctl.T

    def barrier():
        if world > 1:
            torch.distributed.barrier()

    def max_over_ranks(x):
        dev = "cuda" if backend == "nccl" else "cpu"
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        return float(t.item())

    # ---- warm-up (first step eager: counts our launches; then graph capture) ----
    l0 = nat.lib().dp_launch_count()
    runner.step()
    torch.cuda.synchronize()
    launches_per_step = nat.lib().dp_launch_count() - l0
    # N > 1 over NCCL: the library's own communicator enqueues the collectives on
    # the step's stream, so the update is captured with them (gloo: eager)
    use_graph = all(c.xchg is None or c.xchg.capturable for c in ctls) and not args.no_graph
    if use_graph:
        runner.capture()

    def one():
        if use_graph:
            runner._graph.replay()
        else:
            runner.step()

    for _ in range(max(0, args.warmup - 1)):
        one()
    torch.cuda.synchronize()

    # ---- timed region: K steps, L2 flushed between steps, CUDA events ----
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for i in range(args.steps):
            flush.fill_(float(i))
            evs[i][0].record(stream)
            one()
            evs[i][1].record(stream)
        torch.cuda.synchronize()
    barrier()
    step_ms = [s.elapsed_time(e) for s, e in evs]
    tot_ms = sum(step_ms)
    if world > 1:
        tot_ms = max_over_ranks(tot_ms)
    ms_per_step = tot_ms / args.steps
    value = K * args.steps / (tot_ms * 1e-3)
    for c in ctls:
        c.check_errors()

    # ---- phase profile (eager, events at phase boundaries) ----
    phases = {}
    if args.profile_phases > 0 and len(ctls) == 1:
        marks = []

        def mark(name):
            e = torch.cuda.Event(enable_timing=True)
            e.record(stream)
            marks.append((name, e))

        for _ in range(args.profile_phases):
            flush.fill_(0.0)
            marks.clear()
            ctl.step(marks=mark)
            torch.cuda.synchronize()
            for (n0, e0), (_n1, e1) in zip(marks, marks[1:]):
                phases.setdefault(n0, []).append(e0.elapsed_time(e1))
        phases = {k: statistics.mean(v) for k, v in phases.items()}

    # ---- e2e through the public API with host buffers ----
    hp = [torch.empty(st.params.numel(), dtype=torch.float64, pin_memory=True) for st in stores]
    for h, st in zip(hp, stores):
        h.copy_(st.params.cpu())
    ho = [torch.empty_like(h, pin_memory=True) for h in hp]
    hl = [torch.empty(8, dtype=torch.float64, pin_memory=True) for _ in ctls]
    hpl = [torch.empty(c.K_local, c.T, dtype=torch.uint8, pin_memory=True) for c in ctls]
    h2d = sum(h.numel() * 8 for h in hp)
    d2h = h2d + sum(c.K_local * c.T + 64 for c in ctls)
    e2e_ms = []
    for i in range(args.steps):
        flush.fill_(1.0)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(stream)
        for h, st in zip(hp, stores):
            st.params.copy_(h, non_blocking=True)
        one()
        for j, c in enumerate(ctls):
            ho[j].copy_(stores[j].params, non_blocking=True)
            hpl[j].copy_(c.choice, non_blocking=True)
            hl[j].copy_(c.log[:8], non_blocking=True)
        e.record(stream)
        torch.cuda.synchronize()
        e2e_ms.append(s.elapsed_time(e))
        for h, o in zip(hp, ho):
            h.copy_(o)
    e2e_tot = sum(e2e_ms)
    if world > 1:
        e2e_tot = max_over_ranks(e2e_tot)
    e2e_value = K * args.steps / (e2e_tot * 1e-3)

    cert = ctls[0].sampling_certificate()  # collective when sharded: every rank calls it
    if rank != 0:
        if world > 1:
            torch.distributed.destroy_process_group()
        return

    # ---- roofline of the dominant kernel ----
    peak64 = fp64_peak_tflops(nat, torch)
    dom = max(phases, key=phases.get) if phases else "decode"
    # C4 has no per-phase profile: its decoders are timed as the whole round
    dec_ms = phases.get("decode", ms_per_step)
    dec_flops = sum(decoder_flops_per_placement(c.T, c.task.topo.num_devices) * c.K_local for c in ctls)
    pol_flops = sum(policy_flops_per_placement(c.T, c.task.topo.num_devices, c.K) * c.K_local for c in ctls)
    achieved = dec_flops / (dec_ms * 1e-3) / 1e12
    # DRAM bytes per launch from the committed ncu capture of this workload (C3 K=256 or
    # C5 K=4096 on one GPU); other workloads report null rather than another's number
    k_loc = [c.K_local for c in ctls]
    wl = {("C3", 256): "", ("C5", 4096): "_C5"}.get((args.config, k_loc[0] if len(k_loc) == 1 else -1))
    tr = ncu_traffic("dec_kernel", wl) if wl is not None else None
    roofline = {
        "kernel": "dec_kernel (dp_policy_decode)", "bound": "fp64", "achieved": achieved, "peak": peak64,
        "unit": "TFLOP/s", "frac": achieved / peak64 if peak64 else None,
        "traffic": (tr or {}).get("bytes_per_launch"), "traffic_source": (tr or {}).get("source") if tr else
        "none: no committed ncu capture of this workload (C3 K=256 and C5 K=4096 on one GPU have one)",
        "peak_source": "measured fp64 DFMA probe (dp_fp64_fma_probe) on this GPU; MEASURED_PEAKS.json "
                       "has no fp64 figure (bf16 tensor peak is not the denominator of an fp64 kernel)",
        "algorithmic_flops_per_launch": dec_flops, "avg_launch_ms": dec_ms,
        "dominant_phase": dom, "phase_ms": phases,
        "policy_flops_per_step": pol_flops,
    }
    cpu = None
    if world == 1 and not args.skip_cpu:
        try:
            cpu = cpu_baseline(names, [c.K for c in ctls])
        except Exception as ex:  # pragma: no cover
            cpu = {"error": repr(ex)}
    pk = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{args.config}: {CFG_DESC[args.config]}",
                   "k_per_gpu": k_gpu, "global_k": K, "decoder_len": [c.T for c in ctls] if len(ctls) > 1 else T,
                   "parallelism": f"dp{world} (K sharded)",
                   "l2": "flushed between timed steps (256 MiB write)",
                   "cuda_graph": use_graph},
        "steps_per_sec": 1e3 / ms_per_step,
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h,
                "note": "params H2D from pinned host -> full update -> params, placements, log row D2H"},
        "gpu_launches": launches_per_step * args.steps,
        "gpu_launches_per_step": launches_per_step,
        "roofline": roofline,
        "cpu_baseline": cpu,
        "sampling": cert,
        "clocks": clk.summary(),
        "measured_peaks": {k: pk.get(k) for k in ("hbm_gbs", "bf16_tflops")},
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
