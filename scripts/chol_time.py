"""Tile Cholesky time against the tile-row count (lramm_cholqr_pass with a given Gram: Cholesky +
TRSM; the Cholesky kernel alone from the profiler)."""
import ctypes, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, ROOT)
import numpy as np, torch
from torch.profiler import ProfilerActivity, profile
from paper_2405_16917_b200 import _native as N
from paper_2405_16917_b200._device import ptr, stream_handle

dev = torch.device("cuda")
for w in [int(x) for x in (sys.argv[1:] or ["32", "64", "128", "256", "272", "512", "544", "1056"])]:
    m = 64
    g = torch.Generator(device=dev); g.manual_seed(w)
    y = torch.randn(4 * w, w, dtype=torch.float64, device=dev, generator=g)
    G = (y.T @ y).contiguous()
    yy = torch.randn(m, w, dtype=torch.float64, device=dev, generator=g)
    q = torch.empty(m, w, dtype=torch.float64, device=dev)
    L = torch.empty(w, w, dtype=torch.float64, device=dev)
    info = torch.zeros(4, dtype=torch.int32, device=dev)
    wsz = N.LIB.lramm_cholqr_pass_ws(m, w)
    ws = torch.empty(wsz, dtype=torch.uint8, device=dev)
    call = lambda: N.check(N.LIB.lramm_cholqr_pass(ptr(yy), m, w, w, ptr(G), ptr(q), w, ptr(L), ptr(info), ptr(ws), wsz, stream_handle()))
    for _ in range(3): call()
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(10): call()
        torch.cuda.synchronize()
    t = [ev.device_time for ev in prof.events() if ev.device_type.name == "CUDA" and "chol" in ev.name]
    T = (w + 31) // 32
    print(f"w {w:5d}  T {T:3d}  chol {np.median(t):8.1f} us  per tile row {np.median(t) / T:6.2f} us")
