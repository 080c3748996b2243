"""Per-source-line warp-stall breakdown from an ncu report's source page
(ncu -i X --page source --csv --print-source cuda,sass > file)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
hdr = [r for r in rows if r and r[0] == "Line No"][0]
stall = [(i, h[6:]) for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
cur, out = None, []
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if len(r) > 6 and r[0] not in ("", "Line No") and r[2] == "-":
        try:
            tot = int(r[4])
        except ValueError:
            continue
        br = sorted(((int(r[i]), nm) for i, nm in stall if r[i].isdigit() and int(r[i]) > 0), reverse=True)[:3]
        out.append((tot, cur, r[0], r[1].strip()[:70], br))
T = sum(o[0] for o in out)
print("total samples", T)
for tot, f, ln, src, br in sorted(out, key=lambda o: -o[0])[:n]:
    b = " ".join(f"{nm}:{v}" for v, nm in br)
    print(f"{tot:7d} {100 * tot / T:5.1f}% {f}:{ln:5s} {src:70s} | {b}")
