"""Summarise an ncu launch list (gpu__time_duration.sum) for the LAST full step."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h, data = rows[hi], rows[hi + 1:]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
seq = []
for r in data:
    nm = r[ki]
    for pre in ("void ", "dp::", "(anonymous namespace)::", "<unnamed>::"):
        nm = nm.replace(pre, "")
    nm = nm.split("(")[0]
    seq.append((nm, float(r[vi].replace(",", "")) / 1000.0))
# the step starts at enc_prologue_kernel: take the last occurrence
starts = [i for i, (n, _) in enumerate(seq) if n.startswith("enc_prologue_kernel")]
step = seq[starts[-1]:] if starts else seq
# bench.py's post-run peak probe is not part of the step
step = [x for x in step if not x[0].startswith("fp64_fma_probe_kernel")]
tot = sum(v for _, v in step)
agg = collections.OrderedDict()
for n, v in step:
    agg[n] = agg.get(n, 0.0) + v
print(f"step total {tot:.1f} us over {len(step)} launches")
for n, v in sorted(agg.items(), key=lambda x: -x[1]):
    print(f"{v:10.1f} us  {100 * v / tot:5.1f}%  {n}")
if len(sys.argv) > 2 and sys.argv[2] == "seq":
    print("\nlaunch order:")
    for n, v in step:
        print(f"{v:10.1f} us  {n}")
