"""Time the fp64 small-matrix kernels in isolation (CUDA events) and report Jacobi sweeps."""
import os, sys, ctypes, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import paper_2405_16917_b200 as L
from paper_2405_16917_b200 import _native as N
from paper_2405_16917_b200._device import WORKSPACE, ptr, stream_handle
dev = torch.device("cuda")
def timeit(fn, reps=5):
    fn(); torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / reps
for (m, n) in [(300, 74), (1000, 138), (4096, 272), (8192, 544)]:
    a = torch.randn(m, n, dtype=torch.float64, device=dev)
    u = torch.empty(m, n, dtype=torch.float64, device=dev); s = torch.empty(n, dtype=torch.float64, device=dev); v = torch.empty(n, n, dtype=torch.float64, device=dev)
    info = torch.zeros(4, dtype=torch.int32, device=dev)
    wsz = N.LIB.lramm_svd_ws(m, n); ws = WORKSPACE.get(wsz, dev)
    f = lambda: N.check(N.LIB.lramm_svd(ptr(a), m, n, ptr(u), ptr(s), ptr(v), ptr(info), ptr(ws), wsz, stream_handle()))
    t = timeit(f, 2)
    sref = torch.linalg.svdvals(a).cpu().numpy()
    print(f"svd {m}x{n}: {t:.3f} ms  sweeps={int(info[0])}  serr={np.max(np.abs(s.cpu().numpy()-sref))/sref[0]:.2e}", flush=True)
    q = torch.empty_like(a); r = torch.empty(n, n, dtype=torch.float64, device=dev)
    wsz = N.LIB.lramm_qr_ws(m, n); ws = WORKSPACE.get(wsz, dev)
    f = lambda: N.check(N.LIB.lramm_qr(ptr(a), m, n, n, ptr(q), n, ptr(r), ptr(ws), wsz, stream_handle()))
    t = timeit(f, 3)
    rr = r.cpu().numpy(); rref = np.linalg.qr(a.cpu().numpy())[1]; sg = np.sign(np.diag(rref))
    print(f"qr  {m}x{n}: {t:.3f} ms  R err={np.max(np.abs(rr - rref*sg[:,None]))/np.max(np.abs(rref)):.2e}", flush=True)
