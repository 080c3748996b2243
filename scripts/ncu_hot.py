"""Summarise an ncu report: top SASS instructions by warp-stall samples, with the
dominant stall reasons (reads `ncu --page source --csv` output)."""
import csv
import subprocess
import sys
from collections import Counter


def main(rep, top=25):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout.splitlines()
    rows = list(csv.reader(out[1:]))
    h = rows[0]
    si = h.index("Warp Stall Sampling (All Samples)")
    stall_cols = [i for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
    tot = 0
    recs = []
    by_reason = Counter()
    for r in rows[1:]:
        if len(r) < len(h):
            continue
        s = int(r[si] or 0)
        tot += s
        reasons = {h[i]: int(r[i] or 0) for i in stall_cols}
        by_reason.update(reasons)
        recs.append((s, r[0], r[1].strip(), reasons))
    recs.sort(reverse=True)
    print(f"total samples {tot}")
    print("by reason:", ", ".join(f"{k[6:]}={v * 100 / max(tot, 1):.1f}%" for k, v in by_reason.most_common(8)))
    for s, addr, src, reasons in recs[:top]:
        rs = ", ".join(f"{k[6:]}:{v}" for k, v in Counter(reasons).most_common(3) if v)
        print(f"{s * 100 / max(tot, 1):5.1f}%  {addr[-5:]}  {src[:60]:60s} {rs}")


def lines(rep, top=30):
    """Aggregate stall samples per CUDA source line (needs -lineinfo)."""
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout.splitlines()
    cur_file, cur = "", None
    agg = Counter()
    text = {}
    hdr = None
    for r in csv.reader(out):
        if not r:
            continue
        if r[0] == "File Path":
            cur_file = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) < 5:
            continue
        if r[0]:
            cur = (cur_file, int(r[0]))
            text[cur] = r[1].strip()
            continue
        try:
            s = int(r[4])
        except ValueError:
            continue
        if cur:
            agg[cur] += s
    tot = sum(agg.values())
    print(f"total samples {tot}")
    for (f, ln), s in agg.most_common(top):
        print(f"{s * 100 / max(tot, 1):5.1f}%  {f}:{ln:<5d} {text[(f, ln)][:90]}")


if __name__ == "__main__":
    if len(sys.argv) > 2 and sys.argv[2] == "lines":
        lines(sys.argv[1], int(sys.argv[3]) if len(sys.argv) > 3 else 30)
    else:
        main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
