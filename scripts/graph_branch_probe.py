"""How a CUDA graph with two independent branches starts them: two streams, N small kernels each,
captured (a) branch after branch, (b) interleaved; start time of each branch in one replay."""
import torch
from torch.profiler import ProfilerActivity, profile

N = 150
dev = torch.device("cuda")
xa = torch.zeros(1 << 16, device=dev)
xb = torch.zeros(1 << 16, device=dev)
for mode in ("sequential", "interleaved"):
    s0 = torch.cuda.Stream()
    s1 = torch.cuda.Stream()
    cap = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    torch.cuda.synchronize()
    with torch.cuda.stream(cap):
        with torch.cuda.graph(g, stream=cap):
            s0.wait_stream(cap)
            s1.wait_stream(cap)
            if mode == "sequential":
                with torch.cuda.stream(s0):
                    for _ in range(N):
                        xa.add_(1.0)
                with torch.cuda.stream(s1):
                    for _ in range(N):
                        xb.mul_(1.0)
            else:
                for _ in range(N):
                    with torch.cuda.stream(s0):
                        xa.add_(1.0)
                    with torch.cuda.stream(s1):
                        xb.mul_(1.0)
            cap.wait_stream(s0)
            cap.wait_stream(s1)
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        g.replay()
        torch.cuda.synchronize()
    ev = [e for e in prof.events() if e.device_type.name == "CUDA"]
    t0 = min(e.time_range.start for e in ev)
    by = {}
    for e in ev:
        by.setdefault(getattr(e, "device_resource_id", 0), []).append(e)
    for sid, sel in sorted(by.items()):
        print(mode, "stream", sid, "first start", round(min(e.time_range.start for e in sel) - t0, 1),
              "us, last end", round(max(e.time_range.end for e in sel) - t0, 1), "us, n", len(sel))

# (c) one graph per branch, replayed on two streams; (d) the two branch graphs as child nodes of a parent
s0 = torch.cuda.Stream()
s1 = torch.cuda.Stream()
ga, gb = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
torch.cuda.synchronize()
with torch.cuda.stream(s0):
    with torch.cuda.graph(ga, stream=s0):
        for _ in range(N):
            xa.add_(1.0)
with torch.cuda.stream(s1):
    with torch.cuda.graph(gb, stream=s1):
        for _ in range(N):
            xb.mul_(1.0)
torch.cuda.synchronize()


def two():
    cur = torch.cuda.current_stream()
    s0.wait_stream(cur)
    s1.wait_stream(cur)
    with torch.cuda.stream(s0):
        ga.replay()
    with torch.cuda.stream(s1):
        gb.replay()
    cur.wait_stream(s0)
    cur.wait_stream(s1)


for _ in range(3):
    two()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    two()
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type.name == "CUDA"]
t0 = min(e.time_range.start for e in ev)
by = {}
for e in ev:
    by.setdefault(getattr(e, "device_resource_id", 0), []).append(e)
for sid, sel in sorted(by.items()):
    print("two graphs stream", sid, "first start", round(min(e.time_range.start for e in sel) - t0, 1),
          "us, last end", round(max(e.time_range.end for e in sel) - t0, 1), "us, n", len(sel))
