"""Per-phase cycle breakdown of the LSTM backward kernels (block 0) in one eager update at a bench config."""
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
nat.check(nat.lib().dp_debug_lstm_clocks(1, None), "dbg")
ctl.step()
torch.cuda.synchronize()
nat.check(nat.lib().dp_debug_lstm_clocks(0, out), "dbg")
T = len(task.feats)
names = ["elementwise", "barrier 1", "tanh + mat-vec", "barrier 2"]
for which, base in (("encoder (M=1)", 0), ("decoder (M=2)", 4)):
    v = out[base:base + 4]
    tot = sum(v)
    print(f"{name} K={K} T={T} {which}: {tot / T:.0f} cycles/step")
    for n, x in zip(names, v):
        print(f"  {n:16s} {x / T:8.0f} cycles/step  {100 * x / max(tot, 1):5.1f}%")
