"""Small decodes for compute-sanitizer racecheck / synccheck (FAST, DM and
tensor-core-gate decoder variants).  Usage:
  compute-sanitizer --tool racecheck python scripts/racecheck_decoder.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402

from fixtures import cfg  # noqa: E402
import paper_1706_04972_b200 as dp  # noqa: E402
from paper_1706_04972_b200 import _native as nat  # noqa: E402
from paper_1706_04972_b200 import policy as P  # noqa: E402

for name, K, variant in (("C1", 4, 0), ("C3", 3, 0), ("C3", 3, 4), ("C2", 600, 0), ("C2", 8, 0), ("C2", 300, 0), ("C1", 300, 0)):
    gg, topo, _, _ = cfg(name)
    params = dp.trainer.policy_template(gg, topo, dp.TrainerConfig(seed=1))
    feats = P.GroupFeatures.from_grouped(gg, params.spec)
    nat.check(nat.lib().dp_debug_decoder_variant(variant), "variant")
    pl, lp = P.sample_batch(params, feats, np.random.default_rng(3), K)
    g = P.weighted_grad(params, feats, [list(map(int, p)) for p in pl[:2]], np.array([1.0, -0.5]))
    nat.check(nat.lib().dp_debug_decoder_variant(0), "variant")
    print(name, K, variant, float(lp[0]), float(g.abs().sum()))
