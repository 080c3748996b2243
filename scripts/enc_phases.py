"""Per-phase cycle breakdown of the encoder recurrence (thread 0) at a bench config."""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import torch  # noqa: E402

from fixtures import cfg  # noqa: E402
import paper_1706_04972_b200 as dp  # noqa: E402
from paper_1706_04972_b200 import _native as nat  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C3"
gg, topo, _, _ = cfg(name)
params = dp.trainer.policy_template(gg, topo, dp.TrainerConfig())
feats = dp.GroupFeatures.from_grouped(gg, params.spec)
eng = dp.policy.engine_for(params, feats, 8)
pdev = torch.as_tensor(params.to_flat(), device="cuda")
eng.encode(pdev)
torch.cuda.synchronize()
out = (ctypes.c_int64 * 16)()
nat.check(nat.lib().dp_debug_phase_clocks(1, None), "dbg")
eng.encode(pdev)
torch.cuda.synchronize()
nat.check(nat.lib().dp_debug_phase_clocks(0, out), "dbg")
T = len(feats)
names = ["h loads + dots + reduce", "gate activation", "shuffles + cell + tanh + stores", "barrier"]
tot = sum(out[4:8])
print(f"{name} T={T}: {tot / T:.0f} cycles/step")
for n, v in zip(names, out[4:8]):
    print(f"  {n:32s} {v / T:8.0f} cycles/step  {100 * v / tot:5.1f}%")
