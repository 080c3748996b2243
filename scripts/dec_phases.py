"""Per-phase cycle breakdown of the decoder kernel (block 0) at a bench config."""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from fixtures import cfg  # noqa: E402
import paper_1706_04972_b200 as dp  # noqa: E402
from paper_1706_04972_b200 import _native as nat  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C3"
K = int(sys.argv[2]) if len(sys.argv) > 2 else 256
variant = int(sys.argv[3]) if len(sys.argv) > 3 else 0
skip = int(sys.argv[4]) if len(sys.argv) > 4 else 0
nat.check(nat.lib().dp_debug_decoder_variant(variant), "variant")
gg, topo, _, _ = cfg(name)
params = dp.trainer.policy_template(gg, topo, dp.TrainerConfig())
feats = dp.GroupFeatures.from_grouped(gg, params.spec)
eng = dp.policy.engine_for(params, feats, K)
pdev = torch.as_tensor(params.to_flat(), device="cuda")
eng.encode(pdev)
eng.decode(pdev, K, pcg=(1, 3))
torch.cuda.synchronize()
out = (ctypes.c_int64 * 16)()
nat.check(nat.lib().dp_debug_phase_clocks(1 | (skip << 1), None), "dbg")
eng.decode(pdev, K, pcg=(1, 3))
torch.cuda.synchronize()
nat.check(nat.lib().dp_debug_phase_clocks(0, out), "dbg")
wout = (ctypes.c_int64 * 24)()
nat.check(nat.lib().dp_debug_warp_clocks(wout), "wdbg")
T = len(feats)
names = ["A gates+cell", "C scores/softmax/uc/uh/next-g", "E combine+draw"]
tot = sum(out[:3])
print(f"{name} K={K} T={T} variant={variant} skip={skip}: {tot / T:.0f} cycles/step")
for n, v in zip(names, out[:3]):
    print(f"  {n:32s} {v / T:8.0f} cycles/step  {100 * v / tot:5.1f}%")
print("  per-warp phase-end arrival (cycles/step from the phase start; the barrier waits for the max):")
print("  warp        A        C        E")
for w in range(8):
    print(f"  {w:4d} " + " ".join(f"{wout[w * 3 + i] / T:8.0f}" for i in range(3)))
