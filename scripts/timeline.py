"""Per-stream kernel timeline of one lramm step (torch profiler), condensed.

    python scripts/timeline.py c2
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
use_graph = os.environ.get("TIMELINE_GRAPH", "1") == "1"
if use_graph:  # the bench's execution mode: one step captured into a CUDA graph
    cap = torch.cuda.Stream(device=dev)
    cap.wait_stream(torch.cuda.current_stream(dev))
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.stream(cap):
        L.lramm_device(a, b, p)
        torch.cuda.synchronize()
        with torch.cuda.graph(graph, stream=cap):
            L.lramm_device(a, b, p)
    torch.cuda.synchronize()
    for _ in range(3):
        graph.replay()
    torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    if use_graph:
        graph.replay()
    else:
        L.lramm_device(a, b, p)
    torch.cuda.synchronize()
evs = []
for ev in prof.events():
    if ev.device_type.name != "CUDA":
        continue
    nm = ev.name.replace("lramm::(anonymous namespace)::", "").replace("void ", "").split("(")[0][:34]
    evs.append((ev.time_range.start, ev.time_range.end, getattr(ev, "device_resource_id", 0), nm))
t0 = min(e[0] for e in evs)
streams = collections.defaultdict(list)
for s, e, sid, nm in sorted(evs):
    streams[sid].append((s - t0, e - t0, nm))
for sid, lst in streams.items():
    busy = sum(e - s for s, e, _ in lst)
    span = lst[-1][1] - lst[0][0]
    print(f"stream {sid}: {len(lst)} kernels, busy {busy:.0f} us over span {lst[0][0]:.0f}..{lst[-1][1]:.0f} us")
    gaps = [(lst[i + 1][0] - lst[i][1], lst[i][2], lst[i + 1][2], lst[i][1]) for i in range(len(lst) - 1)]
    tot_gap = sum(g for g, *_ in gaps)
    print(f"   idle between kernels {tot_gap:.0f} us; largest gaps:")
    for g, a_, b_, at in sorted(gaps, reverse=True)[:6]:
        print(f"     {g:7.1f} us at {at:7.0f}: after {a_} before {b_}")
    for s, e, nm in lst:
        if e - s > float(os.environ.get("TIMELINE_MIN_US", "80")):
            print(f"   {s:8.0f} .. {e:8.0f}  {e - s:7.0f} us  {nm}")
