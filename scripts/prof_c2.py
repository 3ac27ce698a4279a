"""Warm per-kernel device-time breakdown of one BASELINE-c2 lramm step (torch profiler / CUPTI)."""
import os, sys, collections
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, ROOT)
import torch
from torch.profiler import profile, ProfilerActivity
import paper_2405_16917_b200 as L
n = int(os.environ.get("C2_N", "4096")); mode = os.environ.get("C2_MODE", "fast")
a = torch.randn(n, n, device="cuda", dtype=torch.float32); b = torch.randn(n, n, device="cuda", dtype=torch.float32)
kw = dict(rank=256, bits=(8, 8, 8), power_iters=1, oversample=16, seed=0, out_dtype=torch.float32 and __import__("numpy").float32)
if mode == "fast": kw.update(mode="fast", sketch_bits=8, power_bits=8, proj_bits=8, granularity="row")
p = L.LrammParams(**kw)
for _ in range(3): L.lramm_device(a, b, p)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(5): L.lramm_device(a, b, p)
e.record(); torch.cuda.synchronize(); print(f"step {s.elapsed_time(e)/5:.3f} ms")
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    L.lramm_device(a, b, p); torch.cuda.synchronize()
agg = collections.defaultdict(lambda: [0.0, 0])
for ev in prof.events():
    if ev.device_type.name != "CUDA": continue
    nm = ev.name.replace("lramm::(anonymous namespace)::", "").replace("void ", "").split("(")[0][:50]
    agg[nm][0] += ev.device_time; agg[nm][1] += 1
tot = sum(v[0] for v in agg.values())
print(f"sum of kernel times {tot/1e3:.3f} ms (two streams overlap)")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:22]:
    print(f"{v[0]:10.1f} us {v[1]:4d}x {v[0]/v[1]:9.1f} us/launch  {k}")
