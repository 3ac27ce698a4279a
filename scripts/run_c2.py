"""One warm-up + N timed device-resident LRAMM calls at BASELINE config 2 (for ncu launch lists)."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import paper_2405_16917_b200 as L
n = int(os.environ.get("C2_N", "4096")); reps = int(os.environ.get("C2_REPS", "1"))
mode = os.environ.get("C2_MODE", "fast")
a = torch.randn(n, n, device="cuda", dtype=torch.float32); b = torch.randn(n, n, device="cuda", dtype=torch.float32)
kw = dict(rank=256, bits=(8, 8, 8), power_iters=1, oversample=16, seed=0)
if mode == "fast":
    kw.update(mode="fast", sketch_bits=8, power_bits=8, proj_bits=8, granularity="row")
p = L.LrammParams(**kw)
out, st, t = L.lramm_device(a, b, p, timings=True); torch.cuda.synchronize()
print("warm", t.rsvd_ms, t.gemm3_ms, flush=True)
for i in range(reps):
    out, st, t = L.lramm_device(a, b, p, timings=True)
    print("rsvd %.3f scaling %.3f g1 %.3f g2 %.3f g3 %.3f ms" % (t.rsvd_ms, t.scaling_ms, t.gemm1_ms, t.gemm2_ms, t.gemm3_ms), flush=True)
torch.cuda.synchronize()
