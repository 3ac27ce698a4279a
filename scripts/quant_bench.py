"""Quantiser micro-benchmark: absmax, single quantise (row-major / transposed) and the two-layout
pair at the BASELINE operand sizes, CUDA events, GB/s of algorithmic traffic.

    python scripts/quant_bench.py [rows cols dtype]
"""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch

from paper_2405_16917_b200 import _native as N

vp = ctypes.c_void_p
dev = torch.device("cuda", 0)
CASES = [(131072, 8192, torch.float32), (8192, 8192, torch.float32), (4096, 4096, torch.float32),
         (131072, 1056, torch.float64), (4096, 272, torch.float64)]
if len(sys.argv) > 3:
    CASES = [(int(sys.argv[1]), int(sys.argv[2]), getattr(torch, sys.argv[3]))]


def timed(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps * 1e3  # us


for rows, cols, dt in CASES:
    x = torch.randn(rows, cols, dtype=dt, device=dev)
    code = N.F32 if dt == torch.float32 else N.F64
    es = x.element_size()
    ldr, ldt = (cols + 15) // 16 * 16, (rows + 15) // 16 * 16
    qr = torch.empty((rows, ldr), dtype=torch.int8, device=dev)
    qt = torch.empty((cols, ldt), dtype=torch.int8, device=dev)
    sr = torch.empty(max(rows, cols), dtype=torch.float64, device=dev)
    st = torch.empty(max(rows, cols), dtype=torch.float64, device=dev)
    amax = torch.zeros(max(rows, cols), dtype=torch.float64, device=dev)
    flag = torch.zeros(1, dtype=torch.int32, device=dev)
    wsz = N.LIB.lramm_quantize_ws(rows, cols)
    ws = torch.empty(wsz, dtype=torch.uint8, device=dev)
    strm = vp(torch.cuda.current_stream().cuda_stream)
    nbytes = rows * cols * es
    out = {}
    for gname, g in (("tensor", N.GRAN_TENSOR), ("row", N.GRAN_ROW), ("col", N.GRAN_COL)):
        out[f"absmax/{gname}"] = (timed(lambda: N.check(N.LIB.lramm_absmax(
            vp(x.data_ptr()), code, rows, cols, cols, g, vp(amax.data_ptr()), vp(flag.data_ptr()), strm))), nbytes)
    for tr in (0, 1):
        out[f"quantize/tensor/T{tr}"] = (timed(lambda: N.check(N.LIB.lramm_quantize_amax(
            vp(x.data_ptr()), code, rows, cols, cols, 8, N.GRAN_TENSOR, tr, vp(amax.data_ptr()),
            vp((qt if tr else qr).data_ptr()), N.I8, ldt if tr else ldr, vp(sr.data_ptr()), strm))),
            nbytes + rows * cols)
    for gr, gt in ((N.GRAN_TENSOR, N.GRAN_TENSOR), (N.GRAN_ROW, N.GRAN_COL)):
        out[f"pair/{gr}{gt} (incl absmax)"] = (timed(lambda: N.check(N.LIB.lramm_quantize_pair(
            vp(x.data_ptr()), code, rows, cols, cols, 8, gr, vp(qr.data_ptr()), ldr, vp(sr.data_ptr()), 8, gt,
            vp(qt.data_ptr()), ldt, vp(st.data_ptr()), vp(flag.data_ptr()), vp(ws.data_ptr()), wsz, strm))),
            2 * nbytes + 2 * rows * cols)
    print(f"{rows}x{cols} {dt}  TR={os.environ.get('LRAMM_QTILE_ROWS', '64')}")
    for k, (us, b) in out.items():
        print(f"  {k:28s} {us:9.1f} us  {b / us / 1e3:7.0f} GB/s")
    del x, qr, qt
    torch.cuda.empty_cache()
