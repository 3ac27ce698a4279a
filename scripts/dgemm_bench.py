"""fp64 DMMA GEMM throughput at the CholeskyQR2 / lift shapes (lramm_dgemm C ABI)."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from paper_2405_16917_b200 import _native as N
from paper_2405_16917_b200._device import WORKSPACE, ptr, stream_handle

dev = torch.device("cuda", 0)
def run(trans, M, Nn, K, reps=5):
    a = torch.randn((K, M) if trans else (M, K), dtype=torch.float64, device=dev)
    b = torch.randn(K, Nn, dtype=torch.float64, device=dev)
    c = torch.empty(M, Nn, dtype=torch.float64, device=dev)
    wsz = N.LIB.lramm_dgemm_ws(trans, M, Nn, K)
    ws = WORKSPACE.get(wsz, dev)
    f = lambda: N.check(N.LIB.lramm_dgemm(trans, M, Nn, K, ptr(a), a.stride(0), ptr(b), b.stride(0), ptr(c), Nn, ptr(ws), wsz, stream_handle(dev)))
    f(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): f()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    ref = (a.T if trans else a) @ b
    err = float((c - ref).abs().max() / ref.abs().max())
    print(f"{'TN' if trans else 'NN'} M={M} N={Nn} K={K}: {ms:.3f} ms  {2*M*Nn*K/ms/1e9:.1f} TFLOP/s  err {err:.1e}")
for args in [(1, 1056, 1056, 131072), (0, 131072, 1056, 1056), (0, 131072, 1024, 1056), (1, 272, 272, 4096),
             (0, 4096, 272, 272), (0, 4096, 4096, 4096), (1, 544, 544, 8192), (0, 8192, 544, 544), (0, 544, 544, 544), (1, 272, 272, 272)]:
    run(*args)
# cuBLAS (torch) at the same shapes, for reference
for (t, M, Nn, K) in [(0, 8192, 544, 544), (1, 544, 544, 8192), (0, 544, 544, 544), (0, 4096, 4096, 4096)]:
    a = torch.randn((K, M) if t else (M, K), dtype=torch.float64, device=dev)
    b = torch.randn(K, Nn, dtype=torch.float64, device=dev)
    f = (lambda: a.T @ b) if t else (lambda: a @ b)
    f(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5): f()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(f"cuBLAS {'TN' if t else 'NN'} M={M} N={Nn} K={K}: {ms:.3f} ms  {2*M*Nn*K/ms/1e9:.1f} TFLOP/s")
