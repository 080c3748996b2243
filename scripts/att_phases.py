"""Per-phase cycle breakdown of the attention backward (block 0) in one eager update."""
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
gg, topo, _, _ = cfg(name)
c = dp.TrainerConfig(k=K, total_updates=4, seed=0)
task = dp.trainer._make_task(gg, topo, c)
store = dp.ParameterStore(task.template.to_flat(), max_steps=8)
ctl = dp.trainer.DeviceController(task, store, np.random.SeedSequence(0).spawn(1)[0], 0)
ctl.step()
torch.cuda.synchronize()
out = (ctypes.c_int64 * 8)()
nat.check(nat.lib().dp_debug_att_clocks(1, None), "dbg")
ctl.step()
torch.cuda.synchronize()
nat.check(nat.lib().dp_debug_att_clocks(0, out), "dbg")
names = ["wait + barrier", "DA + ds", "barrier", "dq / dh_ext", "dE|G + dA", "partial stores", "barrier",
         "tile prologue/epilogue"]
tot = sum(out)
print(f"{name} K={K}: {tot} cycles (block 0)")
for n, v in zip(names, out):
    print(f"  {n:24s} {v:10d}  {100 * v / max(tot, 1):5.1f}%")
