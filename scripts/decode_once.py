"""One eager decode at a config (for ncu captures of the decoder variants).
Usage: python scripts/decode_once.py C2 512 [variant]"""
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
K = int(sys.argv[2]) if len(sys.argv) > 2 else 256
nat.check(nat.lib().dp_debug_decoder_variant(int(sys.argv[3]) if len(sys.argv) > 3 else 0), "variant")
gg, topo, _, _ = cfg(name)
params = dp.trainer.policy_template(gg, topo, dp.TrainerConfig())
feats = dp.GroupFeatures.from_grouped(gg, params.spec)
eng = dp.policy.engine_for(params, feats, K)
pdev = torch.as_tensor(params.to_flat(), device="cuda")
eng.encode(pdev)
for _ in range(2):
    eng.decode(pdev, K, pcg=(1, 3))
torch.cuda.synchronize()
