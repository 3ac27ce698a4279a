"""Warm per-kernel device-time breakdown of one lramm step on a bench.py config (torch profiler / CUPTI).

    python scripts/prof_cfg.py c3
"""
import collections
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

import bench
import paper_2405_16917_b200 as L

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
cfg = bench.CONFIGS[name]
dev = torch.device("cuda", 0)
a, b = bench.synth_pair(cfg, 0, dev)
p = L.LrammParams(rank=cfg["rank"], bits=tuple(cfg["bits"]), power_iters=cfg["power_iters"],
                  oversample=cfg["oversample"], seed=0, mode=cfg["mode"], sketch_bits=cfg["sketch_bits"],
                  power_bits=cfg["power_bits"], proj_bits=cfg["proj_bits"], granularity=cfg["granularity"],
                  out_dtype=np.float32)
for _ in range(3):
    L.lramm_device(a, b, p)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(3):
    L.lramm_device(a, b, p)
e.record()
torch.cuda.synchronize()
print(f"{name}: step {s.elapsed_time(e) / 3:.3f} ms")
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    L.lramm_device(a, b, p)
    torch.cuda.synchronize()
agg = collections.defaultdict(lambda: [0.0, 0])
for ev in prof.events():
    if ev.device_type.name != "CUDA":
        continue
    nm = ev.name.replace("lramm::(anonymous namespace)::", "").replace("void ", "").split("(")[0][:60]
    agg[nm][0] += ev.device_time
    agg[nm][1] += 1
tot = sum(v[0] for v in agg.values())
print(f"sum of kernel times {tot / 1e3:.3f} ms (A and B chains overlap on two streams)")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:25]:
    print(f"{v[0]:11.1f} us {v[1]:4d}x {v[0] / v[1]:10.1f} us/launch  {k}")
