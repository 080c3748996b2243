"""Quick K-sim throughput probe (CUDA events; L2 note: graph is L2-resident by design)."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, torch
from fixtures import cfg
import paper_1706_04972_b200.simulator as S

from paper_1706_04972_b200 import _native as nat

variant = int(sys.argv[1]) if len(sys.argv) > 1 else 0  # 0 auto, 1 warp/placement, 2 thread/placement
nat.check(nat.lib().dp_debug_sim_variant(variant), "variant")
res = {}
for name, Ks in (("C1", [8, 256, 4096, 65536]), ("C2", [64, 4096, 32768]), ("C3", [256, 4096, 65536]), ("C5", [512, 4096])):
    gg, topo, _, _ = cfg(name)
    dg = S.device_graph(gg, topo)
    for K in Ks:
        pl = torch.randint(0, topo.num_devices, (K, gg.num_groups), dtype=torch.uint8, device="cuda")
        out = dg.simulate(pl, by_rank=True)
        for _ in range(3):
            dg.simulate(pl, by_rank=True, out=out)
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        it = 10
        s.record()
        for _ in range(it):
            dg.simulate(pl, by_rank=True, out=out)
        e.record(); torch.cuda.synchronize()
        ms = s.elapsed_time(e) / it
        res[f"{name}_K{K}"] = dict(ms=ms, placements_per_s=K / ms * 1e3)
        print(name, K, f"variant={variant}", f"{ms:.3f} ms", f"{K/ms*1e3:,.0f} placements/s", flush=True)
json.dump(res, open(f"gpurun_out/sim_throughput_v{variant}.json", "w"), indent=1)
