"""c4 graph replay timeline: per-stream gaps between consecutive kernels, concurrency histogram."""
import collections, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, ROOT)
import numpy as np, torch
from torch.profiler import ProfilerActivity, profile
import bench
import paper_2405_16917_b200 as L
cfg = bench.CONFIGS["c4"]; dev = torch.device("cuda", 0)
S = int(os.environ.get("BENCH_STREAMS", 8)); P = int(os.environ.get("PAIRS", 64))
pairs = [bench.synth_pair(cfg, j, dev) for j in range(min(P, 16))]
p = L.LrammParams(rank=cfg["rank"], bits=tuple(cfg["bits"]), power_iters=cfg["power_iters"], oversample=cfg["oversample"],
                  seed=0, mode=cfg["mode"], sketch_bits=8, power_bits=8, proj_bits=8, granularity=cfg["granularity"],
                  out_dtype=np.float32)
streams = [torch.cuda.Stream() for _ in range(S)]
outs = [torch.empty(2048, 2048, device=dev) for _ in range(min(P, 16))]
def step():
    cur = torch.cuda.current_stream()
    for s in streams: s.wait_stream(cur)
    for j in range(P):
        with torch.cuda.stream(streams[j % S]):
            a, b = pairs[j % len(pairs)]
            L.lramm_device(a, b, p, out=outs[j % len(outs)])
    for s in streams: cur.wait_stream(s)
for _ in range(2): step()
torch.cuda.synchronize()
cap = torch.cuda.Stream(); cap.wait_stream(torch.cuda.current_stream())
g = torch.cuda.CUDAGraph()
with torch.cuda.stream(cap):
    step(); torch.cuda.synchronize()
    with torch.cuda.graph(g, stream=cap):
        step()
torch.cuda.synchronize()
for _ in range(3): g.replay()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
print(f"streams {S} pairs {P}: graph replay {e0.elapsed_time(e1):.2f} ms")
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    g.replay(); torch.cuda.synchronize()
evs = []
for ev in prof.profiler.kineto_results.events():
    if "CUDA" not in str(ev.device_type()): continue
    s0 = ev.start_ns() / 1e3
    evs.append((s0, s0 + ev.duration_ns() / 1e3, ev.name(), ev.device_resource_id()))
evs.sort()
base, end = evs[0][0], max(e for _, e, _, _ in evs)
print(f"{len(evs)} activities over {(end - base) / 1e3:.2f} ms; sum of durations {sum(e - s for s, e, _, _ in evs) / 1e3:.1f} ms")
per = collections.defaultdict(list)
for s, e, nm, sid in evs: per[sid].append((s, e, nm))
gaps = []
for sid, ks in per.items():
    for (s0, e0_, _), (s1, _, _) in zip(ks, ks[1:]):
        gaps.append(s1 - e0_)
gaps = np.array(gaps)
print(f"{len(per)} streams; gap between consecutive activities of a stream: median {np.median(gaps):.2f} us, mean {gaps.mean():.2f}, "
      f"p90 {np.percentile(gaps, 90):.2f}, p99 {np.percentile(gaps, 99):.2f}; total gap time per stream {gaps.sum() / len(per) / 1e3:.2f} ms")
# concurrency histogram
pts = sorted([(s, 1) for s, e, _, _ in evs] + [(e, -1) for s, e, _, _ in evs])
cur, last, hist = 0, base, collections.Counter()
for t, d in pts:
    hist[cur] += t - last; last = t; cur += d
tot = sum(hist.values())
print("concurrency (activities in flight): " + ", ".join(f"{k}: {100 * v / tot:.0f}%" for k, v in sorted(hist.items()) if v / tot > 0.01))
# launch rate: starts per 100 us window
starts = np.array([s for s, _, _, _ in evs]) - base
h, _ = np.histogram(starts, bins=np.arange(0, end - base + 100, 100))
print(f"activity starts per 100 us: median {np.median(h):.0f}, max {h.max()}  (-> {100 / max(np.median(h), 1):.2f} us per start)")
