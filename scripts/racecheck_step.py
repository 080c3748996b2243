"""One small eager REINFORCE update (encoder, decoder, simulator, epilogue,
both backward passes, Adam) for compute-sanitizer racecheck / synccheck.
Usage: compute-sanitizer --tool racecheck python scripts/racecheck_step.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from fixtures import cfg  # noqa: E402
import paper_1706_04972_b200 as dp  # noqa: E402

for name, K in [tuple(x.split(":")) for x in (sys.argv[1:] or ["C1:6", "C3:4"])]:
    K = int(K)
    gg, topo, _, _ = cfg(name)
    res = dp.train(gg, topo, dp.TrainerConfig(k=K, total_updates=2, seed=3))
    print(name, K, res.log[-1])
