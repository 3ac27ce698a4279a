import os, sys, ctypes
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, ROOT)
import torch
from paper_2405_16917_b200 import _native as N
from paper_2405_16917_b200._device import ptr, stream_handle
M, Nn, K = [int(x) for x in sys.argv[1:4]]; odt = sys.argv[4] if len(sys.argv) > 4 else "f32"
dev = torch.device("cuda")
lda = ((K + 15) // 16) * 16
a = torch.randint(-127, 128, (M, lda), dtype=torch.int8, device=dev); b = torch.randint(-127, 128, (Nn, lda), dtype=torch.int8, device=dev)
out = torch.empty(M, Nn, dtype=torch.float32 if odt == "f32" else (torch.float64 if odt == "f64" else torch.int32), device=dev)
rowmode = len(sys.argv) > 5 and sys.argv[5] == "row"
sa = torch.full((M if rowmode else 1,), 0.37, dtype=torch.float64, device=dev); sb = torch.full((Nn if rowmode else 1,), 1.3, dtype=torch.float64, device=dev)
e = N.Epilogue(); e.out_dtype = {"f32": N.F32, "f64": N.F64, "i32": N.I32}[odt]; e.out = out.data_ptr(); e.ldo = Nn
e.row_scale = sa.data_ptr(); e.col_scale = sb.data_ptr(); e.alpha = 1.0
if rowmode: e.row_scale_inc = 1; e.col_scale_inc = 1
st = stream_handle()
for _ in range(3): N.check(N.LIB.lramm_igemm(M, Nn, K, ptr(a), lda, ptr(b), lda, ctypes.byref(e), 1, st))
torch.cuda.synchronize()
s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s0.record()
for _ in range(10): N.check(N.LIB.lramm_igemm(M, Nn, K, ptr(a), lda, ptr(b), lda, ctypes.byref(e), 1, st))
s1.record(); torch.cuda.synchronize()
us = s0.elapsed_time(s1) / 10 * 1e3
print(f"igemm {M}x{Nn}x{K} -> {odt}{' row/col scales' if rowmode else ''}: {us:.1f} us  {2*M*Nn*K/us/1e6:.1f} TOPS")
