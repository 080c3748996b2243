"""Time the decoder weight-gradient kernels (tcgen05 vs DMMA and ablations) at
C3 K=256: run under `ncu --metrics gpu__time_duration.sum -k regex:dec_wgrad`."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests"))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from fixtures import cfg  # noqa: E402

import paper_1706_04972_b200 as dp  # noqa: E402
from paper_1706_04972_b200 import _native as nat  # noqa: E402
from paper_1706_04972_b200 import policy as P  # noqa: E402

name, K = (sys.argv[1], int(sys.argv[2])) if len(sys.argv) > 2 else ("C3", 256)
modes = [int(x) for x in (sys.argv[3].split(",") if len(sys.argv) > 3 else ["0", "1", "3", "4", "5"])]
gg, topo, _, _ = cfg(name)
params = dp.trainer.policy_template(gg, topo, dp.TrainerConfig(seed=0))
feats = P.GroupFeatures.from_grouped(gg, params.spec)
eng = P.engine_for(params, feats, K)
pdev = torch.as_tensor(params.to_flat(), device=eng.device)
eng.encode(pdev)
eng.decode(pdev, K, pcg=P.generator_state(np.random.default_rng(1)))
eng.backward_rows(pdev, K)
adv = torch.as_tensor(np.random.default_rng(2).normal(size=K), device=eng.device)
for m in modes:
    nat.check(nat.lib().dp_debug_tensor_core(m), "mode")
    for _ in range(3):
        eng.backward_grads(pdev, K, adv)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record()
    for _ in range(20):
        eng.backward_grads(pdev, K, adv)
    ev[1].record()
    torch.cuda.synchronize()
    print(f"mode {m}: grads pass {ev[0].elapsed_time(ev[1]) / 20 * 1000:.1f} us", flush=True)
nat.check(nat.lib().dp_debug_tensor_core(0), "mode")
