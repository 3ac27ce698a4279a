"""Three-stage low-rank quantized approximate GEMM on sm_100a (the reference's
`pipeline.py:22-214` surface).

    E1 = QM(V_r^T W_r, d1)   E2 = QM(E1 Zsc, d2)   E3 = QM(Usc E2, d3)   D = alpha E3 + beta C

`lramm(a, b, params, c)` keeps the reference's signature, validation, error
types and return value `(D, StageTimings)`.  NumPy inputs go through the
host-buffer C entry point `lramm_host_lramm` (host->device copies, the whole
pipeline in one native call, device->host copy of D); CUDA tensors go through the
stream-ordered device entry point `lramm_lramm` and D stays on the device.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from ._device import OMEGA, WORKSPACE, dtype_code, ptr, require_device, stream_handle, to_device_matrix
from .errors import ParameterError, ShapeError
from .quant import _check_bits
from .rsvd import DEFAULT_OVERSAMPLE, native_params, sketch_width

_SEED_TAG_A = 0xA0
_SEED_TAG_B = 0xB0

STAGES = ("rsvd", "scaling", "gemm1", "gemm2", "gemm3")

_PRESETS = {
    "paper-tuned": (8, 4, 8),
    "balanced": (8, 8, 4),
    "max-speed": (4, 4, 4),
}

DEFAULT_D0 = 64


@dataclass(frozen=True)
class LrammParams:
    """Rank, per-stage bit budgets, sketch controls and output scalars (pipeline.py:50-70).

    Extension fields (defaults reproduce the reference):
      mode         "parity": fp64 sketch / power / projection products (the reference);
                   "fast":   those products as int8 tensor-core GEMMs.
      sketch_bits / power_bits / proj_bits   fast-mode bit budgets (default 8).
      granularity  "tensor" (the reference quantiser) or "row" (per-row scales of the
                   left operand, per-column scales of the right operand).
      out_dtype    np.float64 (the reference) or np.float32.
    """

    rank: int
    bits: tuple = (8, 8, 4)
    power_iters: int = 0
    oversample: int = DEFAULT_OVERSAMPLE
    seed: int = 0
    alpha: float = 1.0
    beta: float = 0.0
    mode: str = "parity"
    sketch_bits: int | None = None
    power_bits: int | None = None
    proj_bits: int | None = None
    granularity: str = "tensor"
    out_dtype: object = np.float64

    def __post_init__(self):
        if self.rank < 2:
            raise ParameterError(f"rank must be >= 2, got {self.rank}")
        if len(self.bits) != 3:
            raise ParameterError("bits must be a (d1, d2, d3) triple")
        for d in self.bits:
            _check_bits(d)
        if self.power_iters < 0 or self.oversample < 0:
            raise ParameterError("power_iters and oversample must be >= 0")
        if self.mode not in ("parity", "fast"):
            raise ParameterError(f"mode must be 'parity' or 'fast', got {self.mode!r}")
        if self.granularity not in ("tensor", "row"):
            raise ParameterError(f"granularity must be 'tensor' or 'row', got {self.granularity!r}")
        for name in ("sketch_bits", "power_bits", "proj_bits"):
            v = getattr(self, name)
            if v is not None:
                _check_bits(v, name)
        if np.dtype(self.out_dtype) not in (np.dtype(np.float64), np.dtype(np.float32)):
            raise ParameterError("out_dtype must be float64 or float32")


def preset(name):
    """Named parameter fragment (pipeline.py:73-81)."""
    if name not in _PRESETS:
        raise ParameterError(f"unknown preset {name!r}; choose from {sorted(_PRESETS)}")
    return {"bits": _PRESETS[name], "power_iters": 0, "oversample": DEFAULT_OVERSAMPLE}


@dataclass(frozen=True)
class CostModel:
    """Bit-width-squared weighted MAC counts per pipeline stage (pipeline.py:84-105)."""

    d0: int
    rsvd: int
    scaling: int
    gemm1: int
    gemm2: int
    gemm3: int
    baseline_qgemm: int
    exact_gemm: int

    @property
    def total(self):
        return self.rsvd + self.scaling + self.gemm1 + self.gemm2 + self.gemm3

    def stage_counts(self):
        return {name: getattr(self, name) for name in STAGES}

    def speedup_vs_baseline(self):
        return self.baseline_qgemm / self.total


def cost_model(m, n, k, r, d0=DEFAULT_D0, d1=8, d2=8, d3=8):
    """Weighted MAC counts, formulas kept verbatim from pipeline.py:108-134."""
    if min(m, n, k) < 1 or d0 < 1:
        raise ParameterError("dimensions and d0 must be positive")
    if r < 2:
        raise ParameterError(f"rank must be >= 2, got {r}")
    d0sq, d1sq, d2sq, d3sq = d0 * d0, d1 * d1, d2 * d2, d3 * d3
    return CostModel(
        d0=d0,
        rsvd=round(d0sq * ((m + n) * k * math.log2(r) + (m + n + 2 * k) * r * r)),
        scaling=d0sq * (m * r + n * r),
        gemm1=d0sq * 2 * k * r + d2sq * k * r * r,
        gemm2=d0sq * (r * r + n * r) + d3sq * n * r * r,
        gemm3=d0sq * (n * r + m * r) + d1sq * m * n * r,
        baseline_qgemm=d1sq * m * n * k,
        exact_gemm=d0sq * m * n * k,
    )


@dataclass(frozen=True)
class StageTimings:
    """Per-stage nanoseconds (device time, CUDA events) plus the MAC model (pipeline.py:137-149)."""

    wall_ns: dict
    macs: CostModel

    def wall_total(self):
        return sum(self.wall_ns.values())


def _child_seeds(seed):
    """(seed_A, seed_B) = SeedSequence([seed, 0xA0, 0xB0]).generate_state(2) (pipeline.py:152-156)."""
    state = np.random.SeedSequence(
        [int(seed) & 0xFFFFFFFFFFFFFFFF, _SEED_TAG_A, _SEED_TAG_B]
    ).generate_state(2, dtype=np.uint64)
    return int(state[0]), int(state[1])


def _shape(x, name):
    s = tuple(x.shape) if hasattr(x, "shape") else np.asarray(x).shape
    if len(s) != 2:
        raise ShapeError(f"{name} must be 2-D, got ndim={len(s)}")
    if s[0] < 1 or s[1] < 1:
        raise ShapeError(f"{name} must have positive dimensions, got {s}")
    return s


def _validate(a, b, params, c):
    m, k = _shape(a, "a")
    k2, n = _shape(b, "b")
    if k != k2:
        raise ShapeError(f"inner dimensions differ: {(m, k)} @ {(k2, n)}")
    if c is not None:
        sc = _shape(c, "c")
        if sc != (m, n):
            raise ShapeError(f"c has shape {sc}, expected {(m, n)}")
    if params.rank > min(m, k) or params.rank > min(k, n):
        raise ParameterError(f"rank {params.rank} exceeds operand min dims {min(m, k)}, {min(k, n)}")
    return m, k, n


def _params(params) -> N.Params:
    return native_params(params.rank, params.oversample, params.power_iters, params.bits, params.alpha, params.beta,
                         params.mode, params.sketch_bits, params.power_bits, params.proj_bits, params.granularity)


def _timings_from(t: N.Timings, m, n, k, params) -> StageTimings:
    ms = [t.rsvd_ms, t.scaling_ms, t.gemm1_ms, t.gemm2_ms, t.gemm3_ms]
    d1, d2, d3 = params.bits
    return StageTimings(wall_ns={s: int(round(v * 1e6)) for s, v in zip(STAGES, ms)},
                        macs=cost_model(m, n, k, params.rank, DEFAULT_D0, d1, d2, d3))


def lramm_device(a: torch.Tensor, b: torch.Tensor, params: LrammParams, c: torch.Tensor | None = None,
                 out: torch.Tensor | None = None, timings: bool = False):
    """Device entry (CUDA tensors in, CUDA tensor out, no host synchronisation unless timings)."""
    dev = a.device
    m, k = a.shape
    n = b.shape[1]
    seed_a, seed_b = _child_seeds(params.seed)
    wa = sketch_width((m, k), params.rank, params.oversample)
    wb = sketch_width((k, n), params.rank, params.oversample)
    om_a = OMEGA.device_omega(seed_a, k, wa, dev)
    om_b = OMEGA.device_omega(seed_b, n, wb, dev)
    if a.dtype != b.dtype:  # mixed fp32 / fp64: both in float64, like as_matrix (matcore.py:31-38)
        a, b = a.to(torch.float64), b.to(torch.float64)
    p = _params(params)
    out_t = torch.float64 if np.dtype(params.out_dtype) == np.float64 else torch.float32
    if out is None:
        out = torch.empty((m, n), dtype=out_t, device=dev)
    status = torch.zeros(1, dtype=torch.int32, device=dev)
    wsz = N.LIB.lramm_lramm_ws(m, k, n, ctypes.byref(p))
    ws = WORKSPACE.get(wsz, dev)
    t = N.Timings()
    cc = c if (c is not None and params.beta != 0.0) else None
    N.check(N.LIB.lramm_lramm(ptr(a), ptr(b), dtype_code(a), m, k, n, ctypes.byref(p), ptr(om_a), ptr(om_b), ptr(cc),
                              dtype_code(cc) if cc is not None else N.F64, ptr(out), dtype_code(out), ptr(status),
                              ptr(ws), wsz, ctypes.byref(t) if timings else None, stream_handle(dev)))
    return out, status, t


def lramm(a, b, params, c=None, out=None):
    """Approximate alpha * A @ B + beta * C through the three-stage pipeline (pipeline.py:159-214).

    Returns (D, StageTimings).  Deterministic: identical inputs and params give a
    bitwise identical D.  Extension: ``out`` (C-contiguous, m x n, params.out_dtype)
    receives D, e.g. a pinned host buffer.
    """
    m, k, n = _validate(a, b, params, c)
    d1, d2, d3 = params.bits
    if isinstance(a, torch.Tensor) and a.is_cuda:
        dev = require_device(a.device)
        ta = to_device_matrix(a, dev)
        tb = to_device_matrix(b, dev)
        tc = to_device_matrix(c, dev) if c is not None else None
        out, status, t = lramm_device(ta, tb, params, tc, out=out, timings=True)
        st = int(status.item())
        if st:
            N.check(st)
        return out, _timings_from(t, m, n, k, params)
    # NumPy drop-in: host buffers through the C ABI
    require_device()
    ha = np.asarray(a)
    hb = np.asarray(b)
    in_dt = np.float32 if (ha.dtype == np.float32 and hb.dtype == np.float32) else np.float64
    ha = np.ascontiguousarray(ha, dtype=in_dt)
    hb = np.ascontiguousarray(hb, dtype=in_dt)
    hc = None
    if c is not None and params.beta != 0.0:
        hc = np.ascontiguousarray(c, dtype=np.float64)
    seed_a, seed_b = _child_seeds(params.seed)
    wa = sketch_width((m, k), params.rank, params.oversample)
    wb = sketch_width((k, n), params.rank, params.oversample)
    dev = require_device()
    om_a = OMEGA.device_omega(seed_a, k, wa, dev)  # device-resident: the C ABI uses them in place
    om_b = OMEGA.device_omega(seed_b, n, wb, dev)
    out_dt = np.dtype(params.out_dtype)
    if out is not None:
        if out.shape != (m, n) or out.dtype != out_dt or not out.flags["C_CONTIGUOUS"]:
            raise ShapeError(f"out must be a C-contiguous {(m, n)} {out_dt} array")
        d = out
    else:
        d = np.empty((m, n), dtype=out_dt)
    p = _params(params)
    t = N.Timings()
    vp = lambda x: ctypes.c_void_p(x.ctypes.data) if x is not None else ctypes.c_void_p(0)  # noqa: E731
    rc = N.LIB.lramm_host_lramm(vp(ha), vp(hb), N.F32 if in_dt == np.float32 else N.F64, m, k, n, ctypes.byref(p),
                                ctypes.c_void_p(om_a.data_ptr()), ctypes.c_void_p(om_b.data_ptr()), vp(hc), N.F64, vp(d),
                                N.F32 if out_dt == np.float32 else N.F64,
                                ctypes.byref(t))
    N.check(rc)
    return d, _timings_from(t, m, n, k, params)


def gemm(a, b, alpha=1.0, beta=0.0, c=None):
    """Reference GEMM alpha * A @ B + beta * C in float64 (matcore.py:133-152), on device."""
    from . import kernels

    if isinstance(a, torch.Tensor) and a.is_cuda:
        from .rsvd import _dgemm

        x = a.to(torch.float64).contiguous()
        y = b.to(torch.float64).contiguous()
        if x.shape[1] != y.shape[0]:
            raise ShapeError(f"inner dimensions differ: {tuple(x.shape)} @ {tuple(y.shape)}")
        prod = _dgemm(0, x, y, x.shape[0], y.shape[1], x.shape[1])
    else:
        x = np.ascontiguousarray(a, dtype=np.float64)
        y = np.ascontiguousarray(b, dtype=np.float64)
        if x.shape[1] != y.shape[0]:
            raise ShapeError(f"inner dimensions differ: {x.shape} @ {y.shape}")
        prod = kernels.matmul(x, y)
    if beta != 0.0 and c is not None:
        return alpha * prod + beta * c
    if alpha != 1.0:
        return alpha * prod
    return prod
