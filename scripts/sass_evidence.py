"""Blackwell instruction evidence in the built library, per kernel: tcgen05 MMA
(UTC*MMA), TMEM loads (LDTM), TMA tensor loads (UTMALDG), TMA bulk copies
(UBLKCP), mbarrier ops (SYNCS.*), distributed-shared-memory async stores (STAS) and
cluster barriers (UCGABAR_*), and legacy fp64 tensor-core DMMA.
usage: python scripts/sass_evidence.py [lib.so] > profiles/r02_sass_evidence.txt"""
import collections
import re
import subprocess
import sys

lib = sys.argv[1] if len(sys.argv) > 1 else "paper_1706_04972_b200/_lib/libdevplace_b200.so"
sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
pats = {"UTC*MMA": r"\bUTC[A-Z]*MMA\b", "LDTM": r"\bLDTM\b", "UTMALDG": r"\bUTMALDG\b", "UBLKCP": r"\bUBLKCP\b",
        "SYNCS": r"\bSYNCS\.", "STAS": r"\bSTAS\b", "UCGABAR": r"\bUCGABAR_", "DMMA": r"\bDMMA\b"}
counts = collections.defaultdict(collections.Counter)
fn = None
for line in sass.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        fn = m.group(1)
        continue
    for k, p in pats.items():
        if fn and re.search(p, line):
            counts[fn][k] += 1
names = subprocess.run(["c++filt"], input="\n".join(counts), capture_output=True, text=True).stdout.splitlines()
print(f"# {lib}: kernels with Blackwell async / tensor-core instructions")
print(f"{'kernel':60s} " + " ".join(f"{k:>8s}" for k in pats))
for mangled, nm in sorted(zip(counts, names), key=lambda x: x[1]):
    short = re.sub(r"\(anonymous namespace\)::|dp::|void ", "", nm).split("(")[0]
    print(f"{short[:60]:60s} " + " ".join(f"{counts[mangled][k]:8d}" for k in pats))
