"""Kernel mix of one c4 step (64 pairs on 16 streams), torch profiler."""
import collections, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, ROOT)
import numpy as np, torch
from torch.profiler import ProfilerActivity, profile
import bench
import paper_2405_16917_b200 as L
cfg = bench.CONFIGS["c4"]; dev = torch.device("cuda", 0)
pairs = [bench.synth_pair(cfg, j, dev) for j in range(16)]
p = L.LrammParams(rank=cfg["rank"], bits=tuple(cfg["bits"]), power_iters=cfg["power_iters"], oversample=cfg["oversample"],
                  seed=0, mode=cfg["mode"], sketch_bits=8, power_bits=8, proj_bits=8, granularity=cfg["granularity"],
                  out_dtype=np.float32)
streams = [torch.cuda.Stream() for _ in range(16)]
outs = [torch.empty(2048, 2048, device=dev) for _ in range(16)]
def step():
    cur = torch.cuda.current_stream()
    for s in streams: s.wait_stream(cur)
    for j in range(64):
        with torch.cuda.stream(streams[j % 16]):
            a, b = pairs[j % 16]
            L.lramm_device(a, b, p, out=outs[j % 16])
    for s in streams: cur.wait_stream(s)
for _ in range(2): step()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); step(); e1.record(); torch.cuda.synchronize(); print("eager step %.2f ms" % e0.elapsed_time(e1))
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    step(); torch.cuda.synchronize()
agg = collections.defaultdict(lambda: [0.0, 0])
for ev in prof.events():
    if ev.device_type.name != "CUDA": continue
    nm = ev.name.replace("lramm::(anonymous namespace)::", "").replace("void ", "").split("(")[0][:50]
    agg[nm][0] += ev.device_time; agg[nm][1] += 1
tot = sum(v[0] for v in agg.values())
print("sum of kernel times %.1f ms" % (tot / 1e3))
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:40]:
    print(f"{v[0]:10.0f} us {v[1]:5d}x {v[0]/v[1]:8.1f} us/launch  {k}")
