"""Jacobi SVD probe: accuracy against NumPy and device time of lramm_svd for square widths.

    LRAMM_JACOBI_WB=1 python scripts/jac_wb_check.py [n ...]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch

from paper_2405_16917_b200 import _native as N
from paper_2405_16917_b200._device import WORKSPACE, ptr, stream_handle

dev = torch.device("cuda")
sizes = [int(x) for x in sys.argv[1:]] or [2, 3, 5, 17, 33, 64, 74, 100, 138, 200, 272, 300, 384]
for n in sizes:
    for m in (n, 2 * n + 3):
        g = np.random.default_rng(n * 7 + m)
        q1, _ = np.linalg.qr(g.standard_normal((m, n)))
        q2, _ = np.linalg.qr(g.standard_normal((n, n)))
        sig = np.exp(-np.arange(n) / max(1.0, n / 2.1))
        a_np = (q1 * sig) @ q2.T
        a = torch.tensor(a_np, device=dev)
        u = torch.empty(m, n, dtype=torch.float64, device=dev)
        s = torch.empty(n, dtype=torch.float64, device=dev)
        v = torch.empty(n, n, dtype=torch.float64, device=dev)
        info = torch.zeros(4, dtype=torch.int32, device=dev)
        wsz = N.LIB.lramm_svd_ws(m, n)
        ws = WORKSPACE.get(wsz, dev)
        call = lambda: N.check(N.LIB.lramm_svd(ptr(a), m, n, ptr(u), ptr(s), ptr(v), ptr(info), ptr(ws), wsz,
                                               stream_handle()))
        call()
        torch.cuda.synchronize()
        reps = 5
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            call()
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) / reps * 1e3
        sref = np.linalg.svd(a_np, compute_uv=False)
        sd, ud, vd = s.cpu().numpy(), u.cpu().numpy(), v.cpu().numpy()
        serr = float(np.max(np.abs(sd - sref)) / sref[0])
        orth_u = float(np.max(np.abs(ud.T @ ud - np.eye(n))))
        orth_v = float(np.max(np.abs(vd.T @ vd - np.eye(n))))
        rec = float(np.linalg.norm((ud * sd) @ vd.T - a_np) / np.linalg.norm(a_np))
        ok = serr < 1e-12 and orth_u < 1e-10 and orth_v < 1e-10 and rec < 1e-12
        print(f"m={m:4d} n={n:4d} sweeps={int(info[0]):3d} svd_us={us:9.1f} serr={serr:.1e} orthU={orth_u:.1e} "
              f"orthV={orth_v:.1e} rec={rec:.1e} {'OK' if ok else 'BAD'}", flush=True)

if os.environ.get("JWB_PROFILE"):
    from torch.profiler import ProfilerActivity, profile

    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(3):
            call()
        torch.cuda.synchronize()
    for e in prof.key_averages():
        if e.device_time_total > 0:
            print(f"{e.key[:80]:80s} n={e.count:3d} avg_us={e.device_time_total / e.count:9.1f}")
