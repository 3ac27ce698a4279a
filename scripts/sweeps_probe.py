"""Jacobi sweep counts and SVD time on the projection of a BASELINE config (A side).

    python scripts/sweeps_probe.py c5
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch

import bench
from paper_2405_16917_b200 import _native as N
from paper_2405_16917_b200._device import WORKSPACE, ptr, stream_handle
from paper_2405_16917_b200.rsvd import _qr_device

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
cfg = bench.CONFIGS[name]
dev = torch.device("cuda", 0)
a, _ = bench.synth_pair(cfg, 0, dev)
a = a.double()
w = cfg["rank"] + cfg["oversample"]
om = torch.randn(a.shape[1], w, device=dev, dtype=torch.float64)
q = _qr_device(a @ om)
for _ in range(cfg["power_iters"]):
    q = _qr_device(a @ _qr_device(a.T @ q))
bst = (a.T @ q).contiguous()  # k x w
m, n = bst.shape
u, s, v = (torch.empty(m, n, device=dev, dtype=torch.float64), torch.empty(n, device=dev, dtype=torch.float64),
           torch.empty(n, n, device=dev, dtype=torch.float64))
info = torch.zeros(4, dtype=torch.int32, device=dev)
wsz = N.LIB.lramm_svd_ws(m, n)
ws = WORKSPACE.get(wsz, dev)
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    N.check(N.LIB.lramm_svd(ptr(bst), m, n, ptr(u), ptr(s), ptr(v), ptr(info), ptr(ws), wsz, stream_handle(dev)))
    torch.cuda.synchronize()
    print(f"{name}: BsT {m}x{n} svd {1e3 * (time.perf_counter() - t0):.2f} ms info {info.tolist()}")
sref = torch.linalg.svdvals(bst)
print("sigma rel err", float(((s - sref).abs().max() / sref[0])), "sigma range", float(s[0]), float(s[-1]))
