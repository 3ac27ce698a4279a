import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, ROOT)
import torch
from paper_2405_16917_b200 import _native as N
from paper_2405_16917_b200._device import WORKSPACE, ptr, stream_handle
m, n = int(sys.argv[1]), int(sys.argv[2])
dev = torch.device("cuda")
a = torch.randn(m, n, dtype=torch.float64, device=dev)
u = torch.empty(m, n, dtype=torch.float64, device=dev); s = torch.empty(n, dtype=torch.float64, device=dev); v = torch.empty(n, n, dtype=torch.float64, device=dev)
info = torch.zeros(4, dtype=torch.int32, device=dev)
wsz = N.LIB.lramm_svd_ws(m, n); ws = WORKSPACE.get(wsz, dev)
for _ in range(2):
    N.check(N.LIB.lramm_svd(ptr(a), m, n, ptr(u), ptr(s), ptr(v), ptr(info), ptr(ws), wsz, stream_handle()))
torch.cuda.synchronize(); print("sweeps", int(info[0]))
