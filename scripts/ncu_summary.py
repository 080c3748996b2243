"""Write a compact, committed summary of ncu reports (profiles/<round>_ncu_summary.json + .md).

Per kernel: duration, DRAM bytes (read+write) per launch, SM/memory throughput,
occupancy, IPC, and the top warp-stall reasons from the source page.
"""
import csv
import json
import os
import subprocess
import sys
from collections import Counter

METRICS = {
    "gpu__time_duration.sum": "duration_ns",
    "dram__bytes_read.sum": "dram_read_bytes",
    "dram__bytes_write.sum": "dram_write_bytes",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed": "mem_throughput_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "achieved_occupancy_pct",
    "sm__inst_executed.avg.per_cycle_active": "ipc_per_sm",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active": "fp64_pipe_pct",
    "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active": "dmma_pipe_pct",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum": "smem_wavefronts",
    "launch__registers_per_thread": "registers",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, units, vals = rows[0], rows[1], rows[2]
    scale = {"ns": 1, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6, "s": 1e9, "second": 1e9,
             "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
    d = {}
    for k, name in METRICS.items():
        if k in h:
            v = vals[h.index(k)].replace(",", "")
            try:
                d[name] = float(v) * scale.get(units[h.index(k)], 1)
            except ValueError:
                d[name] = v
    d["kernel"] = vals[h.index("Kernel Name")] if "Kernel Name" in h else "?"
    return d


def stalls(rep, top=6):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout.splitlines()
    rows = list(csv.reader(out[1:]))
    h = rows[0]
    cols = [i for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
    agg = Counter()
    for r in rows[1:]:
        if len(r) < len(h):
            continue
        for i in cols:
            try:
                agg[h[i][6:]] += int(r[i] or 0)
            except ValueError:
                pass
    tot = sum(agg.values()) or 1
    return {k: round(100 * v / tot, 1) for k, v in agg.most_common(top)}


def main(tag, reps):
    os.makedirs("profiles", exist_ok=True)
    res = {}
    for rep in reps:
        if not os.path.exists(rep):
            print(f"skipping {rep}: no report (the kernel did not launch)")
            continue
        name = os.path.basename(rep).replace("prof_", "").replace(".ncu-rep", "")
        d = raw(rep)
        d["stall_pct"] = stalls(rep)
        if "dram_read_bytes" in d and "dram_write_bytes" in d:
            d["dram_bytes_per_launch"] = d["dram_read_bytes"] + d["dram_write_bytes"]
        res[name] = d
    with open(f"profiles/{tag}_ncu_summary.json", "w") as fh:
        json.dump(res, fh, indent=1)
    with open(f"profiles/{tag}_ncu_summary.md", "w") as fh:
        fh.write(f"# ncu --set full summaries ({tag}), one launch each, bench.py {os.environ.get('NCU_WORKLOAD', 'C3 K=256')}\n\n")
        fh.write("| kernel | ms | DRAM MB/launch | SM % | mem % | fp64 pipe % | DMMA pipe % | occ % | IPC/SM | top stalls |\n")
        fh.write("|---|---|---|---|---|---|---|---|---|---|\n")
        for n, d in res.items():
            fh.write(f"| {n} | {d.get('duration_ns', 0) / 1e6:.3f} | {d.get('dram_bytes_per_launch', 0) / 1e6:.1f} | "
                     f"{d.get('sm_throughput_pct', 0):.1f} | {d.get('mem_throughput_pct', 0):.1f} | "
                     f"{d.get('fp64_pipe_pct', 0):.1f} | {d.get('dmma_pipe_pct', 0):.1f} | "
                     f"{d.get('achieved_occupancy_pct', 0):.1f} | {d.get("ipc_per_sm", 0):.2f} | "
                     f"{', '.join(f'{k} {v}%' for k, v in d['stall_pct'].items())} |\n")
    print(json.dumps(res, indent=1)[:3000])


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2:])
