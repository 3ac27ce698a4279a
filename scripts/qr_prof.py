"""Per-kernel device time of one CholeskyQR2 (lramm_qr) at a sketch shape.

    python scripts/qr_prof.py 4096 272
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

from paper_2405_16917_b200 import _native as N
from paper_2405_16917_b200._device import WORKSPACE, ptr, stream_handle

m, n = int(sys.argv[1]), int(sys.argv[2])
dev = torch.device("cuda")
g = torch.Generator(device=dev)
g.manual_seed(1)
u, _ = torch.linalg.qr(torch.randn(m, n, dtype=torch.float64, device=dev, generator=g))
v, _ = torch.linalg.qr(torch.randn(n, n, dtype=torch.float64, device=dev, generator=g))
sig = torch.exp(-torch.arange(n, dtype=torch.float64, device=dev) / (n / 2.1))
a = (u * sig) @ v.T
q = torch.empty_like(a)
r = torch.empty(n, n, dtype=torch.float64, device=dev)
wsz = N.LIB.lramm_qr_ws(m, n)
ws = WORKSPACE.get(wsz, dev)
call = lambda: N.check(N.LIB.lramm_qr(ptr(a), m, n, n, ptr(q), n, ptr(r), ptr(ws), wsz, stream_handle()))
for _ in range(3):
    call()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    call()
e1.record()
torch.cuda.synchronize()
orth = float((q.T @ q - torch.eye(n, device=dev, dtype=torch.float64)).abs().max())
rec = float((q @ r - a).norm() / a.norm())
print(f"qr {m}x{n}: {e0.elapsed_time(e1) / 10 * 1e3:.1f} us/call (stream), orth {orth:.1e}, rec {rec:.1e}")
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(3):
        call()
    torch.cuda.synchronize()
tot = 0.0
for e in sorted(prof.key_averages(), key=lambda e: -e.device_time_total):
    if e.device_time_total > 0:
        tot += e.device_time_total / 3
        print(f"  {e.key[:70]:70s} n={e.count // 3:3d} us/call={e.device_time_total / 3:8.1f}")
print(f"  kernel sum {tot:.1f} us/call")
