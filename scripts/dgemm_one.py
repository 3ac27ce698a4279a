import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, ROOT)
import torch
from paper_2405_16917_b200 import _native as N
from paper_2405_16917_b200._device import WORKSPACE, ptr, stream_handle
trans, M, Nn, K = [int(x) for x in sys.argv[1:5]]
dev = torch.device("cuda", 0)
a = torch.randn((K, M) if trans else (M, K), dtype=torch.float64, device=dev)
b = torch.randn(K, Nn, dtype=torch.float64, device=dev)
c = torch.empty(M, Nn, dtype=torch.float64, device=dev)
wsz = N.LIB.lramm_dgemm_ws(trans, M, Nn, K); ws = WORKSPACE.get(wsz, dev)
for _ in range(5):
    N.check(N.LIB.lramm_dgemm(trans, M, Nn, K, ptr(a), a.stride(0), ptr(b), b.stride(0), ptr(c), Nn, ptr(ws), wsz, stream_handle(dev)))
torch.cuda.synchronize(); print("ok")
