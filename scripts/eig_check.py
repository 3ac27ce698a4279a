"""Device SVD (lramm_svd: CholeskyQR2 + eigen-preconditioned one-sided Jacobi) vs NumPy/LAPACK on
tall matrices shaped like the rsvd projections Bs^T (k x w); prints accuracy and time per call.
    python scripts/eig_check.py            (LRAMM_EIG_PRE=0 for the plain Jacobi path)"""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, ROOT)
import numpy as np
import torch
from paper_2405_16917_b200 import _native as N
from paper_2405_16917_b200._device import WORKSPACE, ptr, stream_handle

rng = np.random.default_rng(7)

def tall(m, n, kind):
    i = np.arange(1, n + 1)
    if kind.startswith("exp:"):
        s = np.exp(-i / float(kind[4:]))
    elif kind.startswith("poly:"):
        s = i ** -float(kind[5:])
    elif kind == "uniform":
        return rng.random((m, n))
    elif kind == "rankdef":
        return rng.standard_normal((m, n // 2)) @ rng.standard_normal((n // 2, n))
    elif kind == "clustered":
        s = np.repeat([1.0, 0.5, 0.25], n // 3 + 1)[:n]
    u, _ = np.linalg.qr(rng.standard_normal((m, n)))
    v, _ = np.linalg.qr(rng.standard_normal((n, n)))
    return (u * s) @ v.T

def run(m, n, kind, reps=int(os.environ.get("EIG_REPS", "20"))):
    a_h = tall(m, n, kind)
    dev = torch.device("cuda")
    a = torch.tensor(a_h, device=dev)
    u = torch.empty(m, n, dtype=torch.float64, device=dev); s = torch.empty(n, dtype=torch.float64, device=dev)
    v = torch.empty(n, n, dtype=torch.float64, device=dev)
    info = torch.zeros(4, dtype=torch.int32, device=dev)
    wsz = N.LIB.lramm_svd_ws(m, n); ws = WORKSPACE.get(wsz, dev)
    call = lambda: N.check(N.LIB.lramm_svd(ptr(a), m, n, ptr(u), ptr(s), ptr(v), ptr(info), ptr(ws), wsz, stream_handle()))
    for _ in range(3):
        call()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        call()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    uu, ss, vt = np.linalg.svd(a_h, full_matrices=False)
    sd, ud, vd = s.cpu().numpy(), u.cpu().numpy(), v.cpu().numpy()
    keep = ss > 1e-12 * ss[0]
    serr = np.max(np.abs(sd[keep] - ss[keep]) / ss[keep])
    r = max(1, int(keep.sum() * 0.9))
    pu = np.linalg.norm(ud[:, :r] @ ud[:, :r].T - uu[:, :r] @ uu[:, :r].T)
    pv = np.linalg.norm(vd[:, :r] @ vd[:, :r].T - vt[:r].T @ vt[:r])
    orth = np.abs(vd.T @ vd - np.eye(n)).max()
    recon = np.linalg.norm((ud * sd) @ vd.T - a_h) / np.linalg.norm(a_h)
    print(f"{m}x{n} {kind:10s} {ms*1e3:9.1f} us  sweeps {int(info[0]):3d}  sig {serr:.1e}  projU {pu:.1e}  projV {pv:.1e}  "
          f"orthV {orth:.1e}  recon {recon:.1e}", flush=True)

cases = [(1024, 74, "exp:32"), (2048, 138, "exp:64"), (4096, 272, "exp:128"), (8192, 544, "poly:1.5"),
         (1000, 300, "uniform"), (600, 200, "rankdef"), (600, 150, "clustered"), (8192, 1056, "exp:256")]
if len(sys.argv) > 1:
    cases = [c for c in cases if c[2] in sys.argv[1:] or str(c[1]) in sys.argv[1:]]
print("LRAMM_EIG_PRE =", os.environ.get("LRAMM_EIG_PRE", "auto"))
for c in cases:
    run(*c)
