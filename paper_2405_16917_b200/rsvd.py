"""Randomised SVD on sm_100a (the reference's `rsvd.py:21-94` surface).

Gaussian range finder with oversampling and power iterations, thin QRs by
CholeskyQR2 (Householder fallback), projection, one-sided Jacobi SVD of the
projected matrix, lift and truncation -- all on device.  Omega is drawn with the
reference's own seeded generator (`rsvd.py:56`, `matcore.py:89-92`) on the host
and cached on the device.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from ._device import OMEGA, WORKSPACE, dtype_code, ptr, require_device, stream_handle, to_device_matrix
from .errors import ParameterError, ShapeError

DEFAULT_OVERSAMPLE = 10
SKETCH_TAG = 0x534B


@dataclass(frozen=True)
class RsvdParams:
    """Rank target, power iteration count, oversampling and sketch seed (rsvd.py:21-36).

    Extension (defaults reproduce the reference): ``mode="fast"`` runs the sketch /
    power / projection products as quantised int8 tensor-core GEMMs at
    ``sketch_bits`` / ``power_bits`` / ``proj_bits`` with ``granularity``
    "tensor" or "row" scales.
    """

    rank: int
    power_iters: int = 0
    oversample: int = DEFAULT_OVERSAMPLE
    seed: int = 0
    mode: str = "parity"
    sketch_bits: int | None = None
    power_bits: int | None = None
    proj_bits: int | None = None
    granularity: str = "tensor"

    def __post_init__(self):
        if self.rank < 1:
            raise ParameterError(f"rank must be >= 1, got {self.rank}")
        if self.power_iters < 0:
            raise ParameterError("power_iters must be >= 0")
        if self.oversample < 0:
            raise ParameterError("oversample must be >= 0")
        if self.mode not in ("parity", "fast"):
            raise ParameterError(f"mode must be 'parity' or 'fast', got {self.mode!r}")
        if self.granularity not in ("tensor", "row"):
            raise ParameterError(f"granularity must be 'tensor' or 'row', got {self.granularity!r}")


@dataclass(frozen=True)
class SvdFactors:
    """Thin SVD triple: u (m x t), sigma (t, descending), v (n x t) (matcore.py:206-229)."""

    u: object
    sigma: object
    v: object

    def __post_init__(self):
        t = self.sigma.shape[0]
        if self.u.shape[1] != t or self.v.shape[1] != t:
            raise ShapeError("factor widths disagree with sigma length")
        s = self.sigma.cpu().numpy() if isinstance(self.sigma, torch.Tensor) else np.asarray(self.sigma)
        if t > 1 and np.any(np.diff(s) > 0):
            raise ParameterError("sigma must be sorted descending")
        if np.any(s < 0):
            raise ParameterError("sigma must be non-negative")

    @property
    def shape(self):
        return (self.u.shape[0], self.v.shape[0])

    def reconstruct(self):
        """Sum of sigma_i u_i v_i^T, shape m x n (device fp64 GEMM)."""
        from .pipeline import gemm

        if isinstance(self.u, torch.Tensor):
            return gemm(self.u * self.sigma, self.v.T.contiguous())
        return gemm(self.u * self.sigma, np.ascontiguousarray(self.v.T))


def sketch_width(shape, rank, oversample):
    """w = min(rank + oversample, min(shape)) (rsvd.py:39-44)."""
    lo = min(shape)
    if rank > lo:
        raise ParameterError(f"rank {rank} exceeds min dim {lo} of {tuple(shape)}")
    return min(rank + oversample, lo)


def native_params(rank, oversample, power_iters, bits=(8, 8, 8), alpha=1.0, beta=0.0, mode="parity",
                  sketch_bits=None, power_bits=None, proj_bits=None, granularity="tensor") -> N.Params:
    p = N.Params()
    p.rank, p.oversample, p.power_iters = int(rank), int(oversample), int(power_iters)
    for i in range(3):
        p.bits[i] = int(bits[i])
    p.alpha, p.beta = float(alpha), float(beta)
    p.mode = N.MODE_FAST if mode == "fast" else N.MODE_PARITY
    p.sketch_bits = int(sketch_bits or 8)
    p.power_bits = int(power_bits or p.sketch_bits)
    p.proj_bits = int(proj_bits or p.power_bits)
    p.granularity = N.GRAN_ROW if granularity == "row" else N.GRAN_TENSOR
    return p


def rsvd_device(x: torch.Tensor, params: RsvdParams):
    dev = x.device
    rows, cols = x.shape
    w = sketch_width((rows, cols), params.rank, params.oversample)
    omega = OMEGA.device_omega(params.seed, cols, w, dev)
    r = params.rank
    p = native_params(r, params.oversample, params.power_iters, mode=params.mode, sketch_bits=params.sketch_bits,
                      power_bits=params.power_bits, proj_bits=params.proj_bits, granularity=params.granularity)
    u = torch.empty((rows, r), dtype=torch.float64, device=dev)
    s = torch.empty(r, dtype=torch.float64, device=dev)
    v = torch.empty((cols, r), dtype=torch.float64, device=dev)
    status = torch.zeros(1, dtype=torch.int32, device=dev)
    wsz = N.LIB.lramm_rsvd_ws(rows, cols, ctypes.byref(p))
    ws = WORKSPACE.get(wsz, dev)
    N.check(N.LIB.lramm_rsvd(ptr(x), dtype_code(x), rows, cols, ctypes.byref(p), ptr(omega), ptr(u), ptr(s), ptr(v),
                             ptr(status), ptr(ws), wsz, stream_handle(dev)))
    st = int(status.item())
    if st:
        N.check(st)
    return u, s, v


def rsvd(a, params):
    """Randomized thin SVD truncated to params.rank (rsvd.py:68-81)."""
    on_dev = isinstance(a, torch.Tensor) and a.is_cuda
    dev = require_device(a.device if on_dev else None)
    x = to_device_matrix(a, dev)
    if x.ndim != 2:
        raise ShapeError(f"matrix must be 2-D, got ndim={x.ndim}")
    u, s, v = rsvd_device(x, params)
    if on_dev:
        return SvdFactors(u=u, sigma=s, v=v)
    return SvdFactors(u=u.cpu().numpy(), sigma=s.cpu().numpy(), v=v.cpu().numpy())


def _qr_device(y: torch.Tensor) -> torch.Tensor:
    m, w = y.shape
    q = torch.empty_like(y)
    wsz = N.LIB.lramm_qr_ws(m, w)
    ws = WORKSPACE.get(wsz, y.device)
    N.check(N.LIB.lramm_qr(ptr(y), m, w, w, ptr(q), w, ctypes.c_void_p(0), ptr(ws), wsz, stream_handle(y.device)))
    return q


def _dgemm(trans_a: int, a: torch.Tensor, b: torch.Tensor, M: int, N_: int, K: int) -> torch.Tensor:
    c = torch.empty((M, N_), dtype=torch.float64, device=a.device)
    wsz = N.LIB.lramm_dgemm_ws(trans_a, M, N_, K)
    ws = WORKSPACE.get(wsz, a.device)
    N.check(N.LIB.lramm_dgemm(trans_a, M, N_, K, ptr(a), a.stride(0), ptr(b), b.stride(0), ptr(c), N_, ptr(ws), wsz,
                              stream_handle(a.device)))
    return c


def range_finder(a, params):
    """Orthonormal Q (m x w) approximating the range of A (rsvd.py:47-65), fp64 products."""
    if params.mode != "parity":
        from .errors import UnsupportedError

        raise UnsupportedError("range_finder exposes the reference (fp64) products; use rsvd/lramm for fast mode")
    on_dev = isinstance(a, torch.Tensor) and a.is_cuda
    dev = require_device(a.device if on_dev else None)
    x = to_device_matrix(a, dev, keep_f32=False)
    m, n = x.shape
    w = sketch_width((m, n), params.rank, params.oversample)
    omega = OMEGA.device_omega(params.seed, n, w, dev)
    y = _dgemm(0, x, omega, m, w, n)
    q = _qr_device(y)
    for _ in range(params.power_iters):
        z = _dgemm(1, x, q, n, w, m)
        qz = _qr_device(z)
        y = _dgemm(0, x, qz, m, w, n)
        q = _qr_device(y)
    return q if on_dev else q.cpu().numpy()


def truncate_svd(factors, rank):
    """Keep the top-`rank` singular triplets (rsvd.py:84-94)."""
    if rank > factors.sigma.shape[0]:
        raise ParameterError(f"rank {rank} exceeds factorization width {factors.sigma.shape[0]}")
    if isinstance(factors.u, torch.Tensor):
        return SvdFactors(u=factors.u[:, :rank].contiguous(), sigma=factors.sigma[:rank].clone(),
                          v=factors.v[:, :rank].contiguous())
    return SvdFactors(u=np.ascontiguousarray(factors.u[:, :rank]), sigma=factors.sigma[:rank].copy(),
                      v=np.ascontiguousarray(factors.v[:, :rank]))


# Size cap of the dense SVD oracle (matcore.py:20-23), read at call time like the reference's
# module constant, so a harness may raise it.
ORACLE_MAX_MIN_DIM = 512


def oracle_svd(a):
    """Dense SVD (matcore.py:232-245) on device: CholeskyQR2 + one-sided Jacobi, capped at
    min(m, n) <= ORACLE_MAX_MIN_DIM (OracleLimitError above it, matcore.py:240-243)."""
    from . import kernels
    from .errors import OracleLimitError

    if isinstance(a, torch.Tensor):
        a = a.detach().cpu().numpy()
    a = np.asarray(a)
    if a.ndim == 2 and min(a.shape) > ORACLE_MAX_MIN_DIM:
        raise OracleLimitError(f"oracle SVD capped at min dim {ORACLE_MAX_MIN_DIM}, got {a.shape}")
    u, s, v = kernels.svd(np.ascontiguousarray(a, dtype=np.float64))
    return SvdFactors(u=u, sigma=s, v=v)
