"""Timeline of pipelined host calls (c3): per stream, the H2D / kernel / D2H phases in time order.

    python scripts/e2e_timeline.py [inflight] [rounds]
"""
import collections, os, sys, threading, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, ROOT)
import numpy as np, torch
from torch.profiler import ProfilerActivity, profile
from concurrent.futures import ThreadPoolExecutor
import bench
import paper_2405_16917_b200 as L

inflight = int(sys.argv[1]) if len(sys.argv) > 1 else 3
rounds = int(sys.argv[2]) if len(sys.argv) > 2 else 3
cfg = bench.CONFIGS[os.environ.get("CFG", "c3")]
dev = torch.device("cuda", 0)
a, b = bench.synth_pair(cfg, 0, dev)
ha = torch.empty(a.shape, dtype=torch.float32, pin_memory=True); ha.copy_(a.cpu())
hb = torch.empty(b.shape, dtype=torch.float32, pin_memory=True); hb.copy_(b.cpu())
ha, hb = ha.numpy(), hb.numpy()
p = L.LrammParams(rank=cfg["rank"], bits=tuple(cfg["bits"]), power_iters=cfg["power_iters"], oversample=cfg["oversample"],
                  seed=0, mode=cfg["mode"], sketch_bits=cfg["sketch_bits"], power_bits=cfg["power_bits"],
                  proj_bits=cfg["proj_bits"], granularity=cfg["granularity"])
tls = threading.local()
def call(_):
    if not hasattr(tls, "out"):
        tls.out = torch.empty((cfg["m"], cfg["n"]), dtype=torch.float64, pin_memory=True).numpy()
    torch.cuda.set_device(0)
    t0 = time.perf_counter()
    L.lramm(ha, hb, p, out=tls.out)
    return (threading.get_ident(), t0, time.perf_counter())
pool = ThreadPoolExecutor(max_workers=inflight)
list(pool.map(call, range(inflight * 2)))
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    T0 = time.perf_counter()
    res = list(pool.map(call, range(inflight * rounds)))
    torch.cuda.synchronize()
    T1 = time.perf_counter()
print(f"{inflight} in flight, {inflight*rounds} calls: {(T1-T0)*1e3/(inflight*rounds):.2f} ms per call")
for tid, t0, t1 in res:
    print(f"  host thread {tid % 10000}: call {1e3*(t0-T0):8.2f} -> {1e3*(t1-T0):8.2f} ms")
evs = []
for ev in prof.profiler.kineto_results.events():
    if "CUDA" not in str(ev.device_type()):
        continue
    nm = ev.name()
    cat = "H2D" if "HtoD" in nm else "D2H" if "DtoH" in nm else "D2D" if "DtoD" in nm else "set" if "emset" in nm else "K"
    s0 = ev.start_ns() / 1e3
    evs.append((s0, s0 + ev.duration_ns() / 1e3, cat, nm, ev.device_resource_id()))
evs.sort()
base = evs[0][0]
print("big copies:")
for s0, e, cat, nm, sid in evs:
    if cat in ("H2D", "D2H") and e - s0 > 500:
        print(f"  {cat} stream {sid:4d} {(s0-base)/1e3:8.2f} -> {(e-base)/1e3:8.2f} ms  ({(e-s0)/1e3:.2f} ms)")
# kernel activity windows per stream (a gap > 1 ms closes a window)
per = collections.defaultdict(list)
for s0, e, cat, nm, sid in evs:
    if cat == "K":
        per[sid].append((s0, e))
print("kernel windows per stream (gap > 1 ms splits):")
rows = []
for sid, ks in per.items():
    cs, ce, busy = ks[0][0], ks[0][1], ks[0][1] - ks[0][0]
    for s0, e in ks[1:]:
        if s0 - ce > 1000:
            rows.append((cs, ce, sid, busy)); cs, ce, busy = s0, e, 0.0
        ce = max(ce, e); busy += e - s0
    rows.append((cs, ce, sid, busy))
for cs, ce, sid, busy in sorted(rows):
    if ce - cs > 200:
        print(f"  stream {sid:4d} {(cs-base)/1e3:8.2f} -> {(ce-base)/1e3:8.2f} ms  (kernel time {busy/1e3:.2f} ms)")
ks = sorted((s0, e) for s0, e, cat, _, _ in evs if cat == "K")
busy = 0.0; cur_s, cur_e = ks[0]
for s0, e in ks[1:]:
    if s0 > cur_e:
        busy += cur_e - cur_s; cur_s, cur_e = s0, e
    else:
        cur_e = max(cur_e, e)
busy += cur_e - cur_s
print(f"kernel-busy union {busy/1e3:.2f} ms of {(evs[-1][1]-base)/1e3:.2f} ms; sum of kernel time {sum(e-s0 for s0,e in ks)/1e3:.2f} ms")
