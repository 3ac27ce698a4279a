"""lramm_svd twice on the same input: outputs must be bitwise identical (no atomics / races)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2405_16917_b200 import _native as N
from paper_2405_16917_b200._device import WORKSPACE, ptr, stream_handle
sys.argv += []
for (m, n) in [(4096, 272), (8192, 544), (8192, 1056), (2048, 138)]:
    g = np.random.default_rng(n)
    a = torch.tensor(g.standard_normal((m, n)) * np.exp(-np.arange(n) / 128.0), device="cuda")
    outs = []
    for rep in range(3):
        u = torch.empty(m, n, dtype=torch.float64, device="cuda"); s = torch.empty(n, dtype=torch.float64, device="cuda")
        v = torch.empty(n, n, dtype=torch.float64, device="cuda"); info = torch.zeros(4, dtype=torch.int32, device="cuda")
        wsz = N.LIB.lramm_svd_ws(m, n); ws = WORKSPACE.get(wsz, torch.device("cuda"))
        N.check(N.LIB.lramm_svd(ptr(a), m, n, ptr(u), ptr(s), ptr(v), ptr(info), ptr(ws), wsz, stream_handle()))
        torch.cuda.synchronize()
        outs.append((u.cpu().numpy(), s.cpu().numpy(), v.cpu().numpy(), int(info[0])))
    same = all(np.array_equal(outs[0][i], o[i]) for o in outs[1:] for i in range(3))
    print(f"{m}x{n}: bitwise identical over 3 runs: {same}  sweeps {[o[3] for o in outs]}", flush=True)
