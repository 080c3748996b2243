import sys, os
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import numpy as np, torch
from fixtures import cfg
import paper_1706_04972_b200 as dp
from paper_1706_04972_b200 import policy as P
which = sys.argv[1]
K = int(sys.argv[2])
gg, topo, _, _ = cfg("C5")
params = dp.trainer.policy_template(gg, topo, dp.TrainerConfig(seed=1))
feats = P.GroupFeatures.from_grouped(gg, params.spec)
if which == "decode":
    pl, lp = P.sample_batch(params, feats, np.random.default_rng(1), K)
    torch.cuda.synchronize(); print("decode ok", lp[:2])
elif which == "step":
    c = dp.TrainerConfig(k=K, total_updates=2, seed=0)
    task = dp.trainer._make_task(gg, topo, c)
    store = dp.ParameterStore(task.template.to_flat(), max_steps=4)
    ctl = dp.trainer.DeviceController(task, store, np.random.SeedSequence(0).spawn(1)[0], 0)
    ctl.step(); torch.cuda.synchronize(); print("step ok")
