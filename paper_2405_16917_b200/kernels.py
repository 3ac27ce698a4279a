"""Drop-in for the reference's kernel plugin `lramm._kernels` (`_kernels/__init__.py:8-39`).

Same four functions, same argument meaning (C-contiguous NumPy buffers in,
fresh NumPy arrays out, inputs never mutated), same errors
(``ValueError("inner dimensions differ")``, ``RuntimeError`` on Jacobi
non-convergence), computed on the B200 through the host-pointer entry points of
liblramm_cuda (include/lramm_cuda.h).  `backend_name()` reports ``"cuda"``.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _native as N
from ._device import require_device

BACKEND = "cuda"


def backend_name():
    return BACKEND


def _vp(a):
    return ctypes.c_void_p(a.ctypes.data)


def _call(rc):
    if rc == N.ERR_SHAPE:
        raise ValueError("inner dimensions differ")
    if rc == N.ERR_NONCONV:
        raise RuntimeError(N.last_error())
    N.check(rc)


def matmul(a, b):
    """Plain float64 product A @ B (_core.pyx:17-32)."""
    if a.shape[1] != b.shape[0]:
        raise ValueError("inner dimensions differ")
    require_device()
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    out = np.empty((a.shape[0], b.shape[1]), dtype=np.float64)
    _call(N.LIB.lramm_host_matmul(_vp(a), _vp(b), _vp(out), a.shape[0], a.shape[1], b.shape[1]))
    return out


def imatmul(a, b):
    """Exact integer product with 64-bit results (_core.pyx:35-50); entries within +-127."""
    if a.shape[1] != b.shape[0]:
        raise ValueError("inner dimensions differ")
    require_device()
    a = np.ascontiguousarray(a, dtype=np.int32)
    b = np.ascontiguousarray(b, dtype=np.int32)
    out = np.empty((a.shape[0], b.shape[1]), dtype=np.int64)
    _call(N.LIB.lramm_host_imatmul(_vp(a), _vp(b), _vp(out), a.shape[0], a.shape[1], b.shape[1]))
    return out


def scale_round_clip(a, scale, cap):
    """Round scale*a to nearest even integer, clamped to [-cap, cap] (_core.pyx:53-69)."""
    require_device()
    a = np.ascontiguousarray(a, dtype=np.float64)
    out = np.empty(a.shape, dtype=np.int32)
    _call(N.LIB.lramm_host_scale_round_clip(_vp(a), a.shape[0], a.shape[1], float(scale), int(cap), _vp(out)))
    return out


def svd(a):
    """Thin SVD (u, sigma descending, v), t = min(m, n) (_jacobi.py:14-50)."""
    require_device()
    a = np.ascontiguousarray(a, dtype=np.float64)
    m, n = a.shape
    t = min(m, n)
    u = np.empty((m, t))
    s = np.empty(t)
    v = np.empty((n, t))
    _call(N.LIB.lramm_host_svd(_vp(a), m, n, _vp(u), _vp(s), _vp(v)))
    return u, s, v
