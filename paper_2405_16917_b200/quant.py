"""Symmetric linear quantiser and integer quantised GEMM on sm_100a.

Same public surface and semantics as the reference's `quant.py`
(`quantize` :55-71, `dequantize` :74-76, `integer_matmul` :79-84, `qgemm` :96-121):
scale = (2^(bits-1)-1) / max|a| in fp64, rint half-to-even, clamp, sentinel
scale 1.0 for all-zero input, dequantisation acc / (sa*sb).  Integer data and
scales are bit-identical to the reference's; products run as int8 tcgen05 GEMMs
with int32 accumulation (bit budgets <= 8), or, for budgets 9..24 and long K, as
8-bit limb products accumulated exactly in int64 (the reference's int64 imatmul).

Inputs may be NumPy arrays (results come back as NumPy, the reference's types)
or CUDA tensors (results stay on the device).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from ._device import WORKSPACE, dtype_code, ptr, require_device, stream_handle, to_device_matrix
from .errors import OverflowRiskError, ParameterError, ShapeError

BITS_MIN = 2
BITS_MAX = 24
MMA_BITS_MAX = 8  # single int8 tensor-core operand; larger budgets use 8-bit limbs


def limbs_for(bits):
    """8-bit limb planes carrying a `bits`-wide integer (1 up to 8 bits, 2 up to 16, 3 up to 24)."""
    return 1 if bits <= 8 else (2 if bits <= 16 else 3)


def bit_cap(bits):
    """Largest representable magnitude for a bit budget: 2^(bits-1) - 1 (quant.py:20-22)."""
    return (1 << (bits - 1)) - 1


def _check_bits(bits, name="bits"):
    if not isinstance(bits, (int, np.integer)) or not BITS_MIN <= int(bits) <= BITS_MAX:
        raise ParameterError(f"{name} must be an integer in [{BITS_MIN}, {BITS_MAX}], got {bits}")
    return int(bits)


@dataclass(frozen=True)
class QuantizedMatrix:
    """Integer matrix plus its quantizer scale and bit budget (quant.py:31-52)."""

    data: object  # int32 (rows, cols): NumPy array or CUDA tensor
    bits: int
    scale: float

    def __post_init__(self):
        if self.data.ndim != 2 or self.data.dtype not in (np.int32, torch.int32):
            raise ShapeError("quantized payload must be a 2-D int32 array")
        _check_bits(self.bits)
        if not self.scale > 0:
            raise ParameterError(f"scale must be positive, got {self.scale}")

    @property
    def rows(self):
        return self.data.shape[0]

    @property
    def cols(self):
        return self.data.shape[1]


def _is_cuda(x) -> bool:
    return isinstance(x, torch.Tensor) and x.is_cuda


def _as_2d(a, name):
    shape = tuple(a.shape) if hasattr(a, "shape") else np.asarray(a).shape
    if len(shape) != 2:
        raise ShapeError(f"{name} must be 2-D, got ndim={len(shape)}")
    if shape[0] < 1 or shape[1] < 1:
        raise ShapeError(f"{name} must have positive dimensions, got {shape}")
    return shape


def quantize_device(x: torch.Tensor, bits: int, granularity: int = N.GRAN_TENSOR, transpose: bool = False,
                    out_dtype: int = N.I8, ld: int | None = None):
    """Device quantiser -> (q tensor, scales fp64 tensor, nonfinite flag tensor)."""
    dev = x.device
    rows, cols = x.shape
    out_rows, out_cols = (cols, rows) if transpose else (rows, cols)
    if ld is None:
        ld = ((out_cols + 15) // 16) * 16 if out_dtype == N.I8 else out_cols
    tdt = {N.I8: torch.int8, N.I32: torch.int32}[out_dtype]
    q = torch.empty((out_rows, ld), dtype=tdt, device=dev)
    nscale = 1 if granularity == N.GRAN_TENSOR else (rows if granularity == N.GRAN_ROW else cols)
    scales = torch.empty(nscale, dtype=torch.float64, device=dev)
    flag = torch.zeros(1, dtype=torch.int32, device=dev)
    wsz = N.LIB.lramm_quantize_ws(rows, cols)
    ws = WORKSPACE.get(wsz, dev)
    N.check(N.LIB.lramm_quantize(ptr(x), dtype_code(x), rows, cols, x.stride(0), int(bits), granularity,
                                 int(transpose), ptr(q), out_dtype, ld, ptr(scales), ptr(flag), ptr(ws), wsz,
                                 stream_handle(dev)))
    return q, scales, flag


def quantize(a, bits):
    """Quantize to `bits`-wide signed integers with a per-matrix scale (quant.py:55-71)."""
    _as_2d(a, "matrix")
    bits = _check_bits(bits)
    on_dev = _is_cuda(a)
    dev = require_device(a.device if on_dev else None)
    x = to_device_matrix(a, dev)
    q, scales, flag = quantize_device(x, bits, N.GRAN_TENSOR, False, N.I32)
    if int(flag.item()):
        raise ParameterError("cannot quantize non-finite entries")
    scale = float(scales.item())
    data = q if on_dev else q.cpu().numpy()
    return QuantizedMatrix(data, bits, scale)


def dequantize(q):
    """Map integers back to float64: entries / scale (quant.py:74-76)."""
    # elementwise true division by a broadcast tensor (a python-scalar divisor is
    # turned into a reciprocal multiply by torch, which is not the reference's rounding)
    if _is_cuda(q.data):
        return q.data.to(torch.float64) / torch.full((1, 1), q.scale, dtype=torch.float64, device=q.data.device)
    dev = require_device()
    d = torch.from_numpy(np.ascontiguousarray(q.data)).to(dev).to(torch.float64)
    return (d / torch.full((1, 1), q.scale, dtype=torch.float64, device=dev)).cpu().numpy()


def _check_overflow(k, bits_a, bits_b):
    # quant.py:87-93: worst-case |sum| = k * cap_a * cap_b must stay below 2^63 (the device path
    # accumulates exactly in int64 whenever int32 would not be enough)
    if k * bit_cap(bits_a) * bit_cap(bits_b) >= 1 << 63:
        raise OverflowRiskError(f"k={k} with bit budgets ({bits_a}, {bits_b}) risks int64 overflow")


def integer_matmul(qa, qb):
    """Exact integer product of two quantized matrices, int64 entries (quant.py:79-84)."""
    if qa.cols != qb.rows:
        raise ShapeError(f"inner dimensions differ: {tuple(qa.data.shape)} @ {tuple(qb.data.shape)}")
    _check_overflow(qa.cols, qa.bits, qb.bits)
    if _is_cuda(qa.data):
        return _imatmul_device(qa.data, qb.data, qa.bits, qb.bits)
    from . import kernels

    a, b = qa.data, qb.data
    return kernels.imatmul(np.ascontiguousarray(a, dtype=np.int32), np.ascontiguousarray(b, dtype=np.int32))


def _imatmul_device(a32: torch.Tensor, b32: torch.Tensor, bits_a: int, bits_b: int) -> torch.Tensor:
    """Exact int64 A . B of device int32 quantised data (entries within +-bit_cap): 8-bit limb
    planes through the tcgen05 kernel, accumulated exactly in int64 (the raw-product epilogue),
    the device counterpart of _kernels.imatmul (_core.pyx:35-50) with no host round trip."""
    dev = a32.device
    m, k = a32.shape
    n = b32.shape[1]
    la, lb = limbs_for(bits_a), limbs_for(bits_b)
    ldk = ((k + 15) // 16) * 16
    ap = torch.zeros((m, ldk), dtype=torch.int32, device=dev)
    ap[:, :k] = a32
    bt = torch.zeros((n, ldk), dtype=torch.int32, device=dev)
    bt[:, :k] = b32.T  # B^T: n x k, K-major
    qa = torch.empty((la, m, ldk), dtype=torch.int8, device=dev)
    qb = torch.empty((lb, n, ldk), dtype=torch.int8, device=dev)
    st = stream_handle(dev)
    N.check(N.LIB.lramm_split_limbs(ptr(ap), m, k, ldk, la, ptr(qa), ldk, st))
    N.check(N.LIB.lramm_split_limbs(ptr(bt), n, k, ldk, lb, ptr(qb), ldk, st))
    out = torch.empty((m, n), dtype=torch.int64, device=dev)
    acc64 = torch.empty((m, n), dtype=torch.int64, device=dev)
    e = N.Epilogue()
    e.out_dtype = N.I64
    e.out = out.data_ptr()
    e.ldo = n
    N.check(N.LIB.lramm_igemm_limbs(m, n, k, ptr(qa), qa.stride(1), qa.stride(0), la, ptr(qb), qb.stride(1),
                                    qb.stride(0), lb, ptr(acc64), ctypes.byref(e), st))
    return out


def qgemm_device(a: torch.Tensor, b: torch.Tensor, bits_a: int, bits_b: int, alpha=1.0, beta=0.0, c=None,
                 out_dtype=torch.float64) -> torch.Tensor:
    """alpha * dequant(int(A) @ int(B)) + beta * C on device; A: m x k, B: k x n."""
    dev = a.device
    m, k = a.shape
    n = b.shape[1]
    la, lb = limbs_for(bits_a), limbs_for(bits_b)
    single = la == 1 and lb == 1 and k * bit_cap(bits_a) * bit_cap(bits_b) < (1 << 31)
    if single:
        qa, sa, fa = quantize_device(a, bits_a, N.GRAN_TENSOR, False, N.I8)
        qb, sb, fb = quantize_device(b, bits_b, N.GRAN_TENSOR, True, N.I8)  # B^T: n x k, K-major
    else:  # reference integers (int32) -> 8-bit limb planes, exact int64 accumulation
        ldk = ((k + 15) // 16) * 16
        qa32, sa, fa = quantize_device(a, bits_a, N.GRAN_TENSOR, False, N.I32, ld=ldk)
        qb32, sb, fb = quantize_device(b, bits_b, N.GRAN_TENSOR, True, N.I32, ld=ldk)
        qa = torch.empty((la, m, ldk), dtype=torch.int8, device=dev)
        qb = torch.empty((lb, n, ldk), dtype=torch.int8, device=dev)
        st = stream_handle(dev)
        N.check(N.LIB.lramm_split_limbs(ptr(qa32), m, k, ldk, la, ptr(qa), ldk, st))
        N.check(N.LIB.lramm_split_limbs(ptr(qb32), n, k, ldk, lb, ptr(qb), ldk, st))
    out = torch.empty((m, n), dtype=out_dtype, device=dev)
    e = N.Epilogue()
    e.out_dtype = N.F64 if out_dtype == torch.float64 else N.F32
    e.out = out.data_ptr()
    e.ldo = n
    e.row_scale = sa.data_ptr()
    e.row_scale_inc = 0
    e.col_scale = sb.data_ptr()
    e.col_scale_inc = 0
    e.alpha = float(alpha)
    e.beta = float(beta) if c is not None else 0.0
    if c is not None:
        e.c = c.data_ptr()
        e.c_dtype = dtype_code(c)
        e.ldc = c.stride(0)
    if single:
        N.check(N.LIB.lramm_igemm(m, n, k, ptr(qa), qa.stride(0), ptr(qb), qb.stride(0), ctypes.byref(e), 1,
                                  stream_handle(dev)))
    else:
        acc64 = torch.empty((m, n), dtype=torch.int64, device=dev)
        N.check(N.LIB.lramm_igemm_limbs(m, n, k, ptr(qa), qa.stride(1), qa.stride(0), la, ptr(qb), qb.stride(1),
                                        qb.stride(0), lb, ptr(acc64), ctypes.byref(e), stream_handle(dev)))
    if int(fa.item()) or int(fb.item()):
        raise ParameterError("cannot quantize non-finite entries")
    return out


def qgemm(a, b, bits_a, bits_b, alpha=1.0, beta=0.0, c=None):
    """Quantized GEMM: alpha * dequant(int(A) @ int(B)) + beta * C (quant.py:96-121)."""
    sa_shape = _as_2d(a, "a")
    sb_shape = _as_2d(b, "b")
    if sa_shape[1] != sb_shape[0]:
        raise ShapeError(f"inner dimensions differ: {sa_shape} @ {sb_shape}")
    if c is not None:
        sc = _as_2d(c, "c")
        if sc != (sa_shape[0], sb_shape[1]):
            raise ShapeError(f"c has shape {sc}, expected {(sa_shape[0], sb_shape[1])}")
    bits_a = _check_bits(bits_a, "bits_a")
    bits_b = _check_bits(bits_b, "bits_b")
    _check_overflow(sa_shape[1], bits_a, bits_b)
    on_dev = _is_cuda(a)
    dev = require_device(a.device if on_dev else None)
    ta = to_device_matrix(a, dev)
    tb = to_device_matrix(b, dev)
    tc = to_device_matrix(c, dev) if (c is not None and beta != 0.0) else None
    out = qgemm_device(ta, tb, bits_a, bits_b, alpha, beta, tc)
    return out if on_dev else out.cpu().numpy()
