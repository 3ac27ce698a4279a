"""Measurement report around the approximate product.

Mirrors the reference's report path: `pipeline.evaluate` / `combined_bound` /
`leading_sigmas` / `ErrorReport` (`pipeline.py:221-328`) and the closed-form bounds of
`bounds.py` (the paper's per-stage error caps, restated as the formulas they document),
plus `rsvd.quantized_svd_approx` (`rsvd.py:97-113`).  The heavy parts run on the device:
the exact product is the fp64 DMMA GEMM (`lramm_dgemm`), singular values come from the
device SVD (`lramm_svd`) or the device randomised SVD, norms are device reductions.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from .errors import ParameterError, ShapeError
from .pipeline import CostModel, LrammParams, gemm, lramm
from .quant import bit_cap, dequantize, quantize
from .rsvd import RsvdParams, oracle_svd, rsvd, truncate_svd



# ------------------------------------------------------------------ bounds (bounds.py)


@dataclass(frozen=True)
class BoundInputs:
    """Sizes, leading / tail singular values and bit budgets of C = A @ B (bounds.py:21-52)."""

    m: int
    n: int
    k: int = 0
    r: int = 0
    sigma1: float = 0.0
    sigma_r1: float = 0.0
    gamma1: float = 0.0
    gamma_r1: float = 0.0
    d1: int = 8
    d2: int = 8
    d3: int = 8
    q: int = 0
    lambda1: float = 0.0
    lambda2: float = 0.0

    def __post_init__(self):
        if self.m < 1 or self.n < 1:
            raise ParameterError("dimensions must be positive")
        if self.sigma1 < self.sigma_r1 or self.sigma_r1 < 0:
            raise ParameterError("need sigma1 >= sigma_r1 >= 0")
        if self.gamma1 < self.gamma_r1 or self.gamma_r1 < 0:
            raise ParameterError("need gamma1 >= gamma_r1 >= 0")


def quant_scalar_var_bound(max_abs, bits):
    """Variance of the scalar quantiser on [-M, M]: M^2 / D^2."""
    if max_abs < 0:
        raise ParameterError("max_abs must be >= 0")
    return max_abs ** 2 / bit_cap(bits) ** 2


def quant_matrix_bound(m, n, scale):
    """Frobenius cap of a whole-matrix quantisation: sqrt(mn) / scale."""
    if scale <= 0:
        raise ParameterError("scale must be positive")
    return math.sqrt(m * n) / scale


def qgemm_bound(bi):
    """Quantised product cap k (sigma1 sqrt(n)/l2 + gamma1 sqrt(m)/l1 + sqrt(mn)/(l1 l2))."""
    if bi.lambda1 <= 0 or bi.lambda2 <= 0:
        raise ParameterError("quantizer scales must be positive")
    root_mn = math.sqrt(bi.m * bi.n)
    return bi.k * (bi.sigma1 * math.sqrt(bi.n) / bi.lambda2 + bi.gamma1 * math.sqrt(bi.m) / bi.lambda1
                   + root_mn / (bi.lambda1 * bi.lambda2))


def svd_trunc_bound(sigma_r1, p, r):
    """Rank-r truncation cap sigma_{r+1} sqrt(p - r)."""
    if r >= p:
        raise ParameterError(f"need r < p, got r={r}, p={p}")
    return sigma_r1 * math.sqrt(p - r)


def rsvd_error_bound(sigma_r1, p, r, q):
    """Randomised rank-r spectral cap (1 + 4 sqrt(2p/(r-1)))^(1/(2q+1)) sigma_{r+1}."""
    if r < 2:
        raise ParameterError(f"bound needs r >= 2, got {r}")
    return (1.0 + 4.0 * math.sqrt(2.0 * p / (r - 1))) ** (1.0 / (2 * q + 1)) * sigma_r1


def _factor_sq_cap(tail, lead, rows, cols, r, cap_left, cap_right):
    """Squared-error cap of a rank-r factorisation of a rows x cols matrix whose scaled left
    factor is quantised with integer cap cap_left and right factor with cap_right."""
    cl, cr = cap_left ** 2, cap_right ** 2
    lead_sq = lead ** 2
    return (tail ** 2 * (cols - r) + rows * r * lead_sq / cl + cols * r * lead_sq / cr
            + rows * cols * r * lead_sq / (cl * cr))


def qsvd_bound(bi):
    """Squared-error cap of a quantised rank-r factorisation of an m x n matrix (bounds.py:101-116)."""
    return _factor_sq_cap(bi.sigma_r1, bi.sigma1, bi.m, bi.n, bi.r, bit_cap(bi.d1), bit_cap(bi.d2))


def _l1(bi):
    # A (m x k): left factor at d1, right at d2, tail over k - r columns
    return _factor_sq_cap(bi.sigma_r1, bi.sigma1, bi.m, bi.k, bi.r, bit_cap(bi.d1), bit_cap(bi.d2))


def _l2(bi):
    # B (k x n): k-side factor at d3, n-side at d2, tail over k - r
    d2c, d3c = bit_cap(bi.d2) ** 2, bit_cap(bi.d3) ** 2
    g1sq = bi.gamma1 ** 2
    return (bi.gamma_r1 ** 2 * (bi.k - bi.r) + bi.k * bi.r * g1sq / d3c + bi.n * bi.r * g1sq / d2c
            + bi.k * bi.n * bi.r * g1sq / (d2c * d3c))


def lramm_general_bound(bi):
    """sqrt(L1 L4) + sqrt(L2 L3) + sqrt(L1 L2), L3 = sigma1^2 k, L4 = gamma1^2 k (bounds.py:145-157)."""
    l1, l2 = _l1(bi), _l2(bi)
    l3, l4 = bi.sigma1 ** 2 * bi.k, bi.gamma1 ** 2 * bi.k
    return math.sqrt(l1 * l4) + math.sqrt(l2 * l3) + math.sqrt(l1 * l2)


def lramm_specific_bound(k, r, sigma1, f_r, d1_cap, d2_cap, d3_cap):
    """Symmetric-case cap k s1^2 sqrt(r) (P + Q) + k r s1^2 P Q (bounds.py:160-174)."""
    if f_r < 0:
        raise ParameterError("f_r must be >= 0")
    p = math.sqrt(f_r + 1.0 / d1_cap + 1.0 / d2_cap + k / (d1_cap * d2_cap))
    q = math.sqrt(f_r + 1.0 / d2_cap + 1.0 / d3_cap + k / (d2_cap * d3_cap))
    s1sq = sigma1 ** 2
    return k * s1sq * math.sqrt(r) * (p + q) + k * r * s1sq * p * q


def spectrum_shape_factor(sigma1, sigma_r1, k, r):
    """f(r) = (sigma_{r+1} / sigma_1)^2 (k - r)."""
    if sigma1 <= 0:
        raise ParameterError("sigma1 must be positive")
    return (sigma_r1 / sigma1) ** 2 * (k - r)


# ------------------------------------------------------------------ report (pipeline.py:221-328)


@dataclass(frozen=True)
class ErrorReport:
    """Measured errors of one approximate multiply plus the matching bound."""

    m: int
    n: int
    k: int
    r: int
    d1: int
    d2: int
    d3: int
    q: int
    seed: int
    fro_error: float
    rel_error: float
    bound_combined: float
    macs: CostModel
    wall_ns: dict
    sigma_source: str = "oracle"

    def to_dict(self):
        macs = self.macs.stage_counts()
        macs["total"] = self.macs.total
        return {"m": self.m, "n": self.n, "k": self.k, "r": self.r, "d1": self.d1, "d2": self.d2, "d3": self.d3,
                "q": self.q, "seed": self.seed, "fro_error": self.fro_error, "rel_error": self.rel_error,
                "bound_combined": self.bound_combined, "macs": macs, "wall_ns": dict(self.wall_ns),
                "sigma_source": self.sigma_source}


def _shape(a):
    return tuple(a.shape)


def leading_sigmas(a, count, seed=0):
    """First `count` singular values and their source: the device SVD ('oracle') up to the
    reference's oracle cap, else the device randomised SVD ('rsvd') (pipeline.py:263-274)."""
    shape = _shape(a)
    if len(shape) != 2:
        raise ShapeError("matrix must be 2-D")
    import sys

    _rsvd = sys.modules[__package__ + ".rsvd"]  # the module (the package re-exports the function); cap read at call time (matcore.py:23)

    if min(shape) <= _rsvd.ORACLE_MAX_MIN_DIM:
        return np.asarray(oracle_svd(a).sigma)[:count], "oracle"
    f = rsvd(a, RsvdParams(rank=min(count, min(shape)), power_iters=1, seed=seed))
    return np.asarray(f.sigma)[:count], "rsvd"


def combined_bound(a, b, params: LrammParams):
    """`lramm_general_bound` from measured singular values (pipeline.py:277-297)."""
    r = params.rank
    sa, src_a = leading_sigmas(a, r + 1, params.seed)
    sb, src_b = leading_sigmas(b, r + 1, params.seed + 1)
    d1, d2, d3 = params.bits
    bi = BoundInputs(m=_shape(a)[0], n=_shape(b)[1], k=_shape(a)[1], r=r, sigma1=float(sa[0]),
                     sigma_r1=float(sa[r]) if len(sa) > r else 0.0, gamma1=float(sb[0]),
                     gamma_r1=float(sb[r]) if len(sb) > r else 0.0, d1=d1, d2=d2, d3=d3, q=params.power_iters)
    source = "oracle" if (src_a == "oracle" and src_b == "oracle") else "rsvd"
    return lramm_general_bound(bi), source


def _fro(x):
    t = x if isinstance(x, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64)).cuda()
    return float(torch.linalg.vector_norm(t.to(torch.float64)).item())


def frobenius_norm(a):
    """sqrt of the sum of squared entries (matcore.py:155-158), reduced on the device."""
    if len(_shape(a)) != 2:
        raise ShapeError("matrix must be 2-D")
    return _fro(a)


def relative_error(approx, exact):
    """||approx - exact||_F / ||exact||_F (matcore.py:190-199)."""
    if _shape(approx) != _shape(exact):
        raise ShapeError(f"shape mismatch: {_shape(approx)} vs {_shape(exact)}")
    dev = lambda x: (x if isinstance(x, torch.Tensor) else  # noqa: E731
                     torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64))).cuda().to(torch.float64)
    ta, te = dev(approx), dev(exact)
    denom = _fro(te)
    if denom == 0.0:
        from .errors import DegenerateDenominatorError

        raise DegenerateDenominatorError("exact matrix has zero Frobenius norm")
    return _fro(ta - te) / denom


def evaluate(a, b, params: LrammParams, c=None):
    """Run the pipeline, compare with the exact product on the device, attach the bound
    (pipeline.py:300-328).  Returns (D, ErrorReport)."""
    d, timings = lramm(a, b, params, c=c)
    exact = gemm(a, b, params.alpha, params.beta, c)
    dd = d if isinstance(d, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(d, dtype=np.float64)).cuda()
    ee = exact if isinstance(exact, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(exact)).cuda()
    ee = ee.to(dd.device, torch.float64)
    fro = _fro(dd.to(torch.float64) - ee)
    denom = _fro(ee)
    if denom == 0.0:  # matcore.relative_error (matcore.py:196-198), called by evaluate (pipeline.py:308)
        from .errors import DegenerateDenominatorError

        raise DegenerateDenominatorError("exact matrix has zero Frobenius norm")
    rel = fro / denom
    bound, source = combined_bound(a, b, params)
    d1, d2, d3 = params.bits
    m, k = _shape(a)
    report = ErrorReport(m=m, n=_shape(b)[1], k=k, r=params.rank, d1=d1, d2=d2, d3=d3, q=params.power_iters,
                         seed=params.seed, fro_error=fro, rel_error=rel, bound_combined=bound,
                         macs=timings.macs, wall_ns=timings.wall_ns, sigma_source=source)
    return d, report


def quantized_svd_approx(a, rank, bits_u, bits_v):
    """Rank-`rank` approximation with both factors quantised (rsvd.py:97-113): the singular-value
    scaled U_r at bits_u and V_r at bits_v; returns (QU, QV, dequant(QU) dequant(QV)^T)."""
    shape = _shape(a)
    if rank > min(shape):
        raise ParameterError(f"rank {rank} exceeds min dim {min(shape)}")
    f = truncate_svd(oracle_svd(a), rank)
    u = np.asarray(f.u) * np.asarray(f.sigma)
    qu = quantize(np.ascontiguousarray(u), bits_u)
    qv = quantize(np.ascontiguousarray(np.asarray(f.v)), bits_v)
    rec = gemm(dequantize(qu), np.ascontiguousarray(dequantize(qv).T))
    return qu, qv, rec
