"""CPU ORACLE for the LRAMM approximate-GEMM hot path -- TEST INFRASTRUCTURE ONLY.

This module is a NumPy restatement of the reference algorithm
(`/root/reference/pkg/src/lramm`, arXiv 2405.16917 Algorithm 3).  It is the
*checker*: only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s
`cpu_baseline` / `--impl reference` legs may import it.  The product package
(`paper_2405_16917_b200`) never imports, links or executes anything in
`oracle/`; it fails loudly when its CUDA library is missing.

Pinning.  The restatement is pinned two ways (see `tests/test_oracle_golden.py`):
  * the reference's own known-answer tests for this path
    (`pkg/tests/test_quant.py:32-47`, `test_backends.py:41-51`, ...) are
    re-asserted against it;
  * golden vectors produced by running the *unmodified reference* in the build
    container (`tests/golden/make_golden.py`, reference installed into
    `oracle/_ref` by `oracle/build_ref.sh`) must be reproduced: integer data and
    scales bit-exactly, `lramm()` outputs to <= 1e-12 relative Frobenius
    (the reference's own compiled-vs-pure backend floor is 1.7e-13).

Two execution modes:
  * ``mode="parity"`` -- the reference algorithm itself: fp64 sketch /
    projection products, Householder QR, dense SVD, then the three per-tensor
    quantized recombination products (`pipeline.py:159-214`).
  * ``mode="fast"`` -- the BASELINE extension: the sketch (Y = X.Omega), power
    (X^T.Q, X.Qz) and projection (Q^T.X) products are run as quantized integer
    GEMMs at ``sketch_bits`` / ``power_bits`` / ``proj_bits`` with per-tensor or
    per-row scales; everything that is re-quantized downstream stays fp64.
    The quantizer is the reference's (`quant.py:55-71`) applied per tensor, per
    row or per column; the dequantization mirrors `quant.py:116`.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

# --------------------------------------------------------------------------
# constants mirrored from the reference

BITS_MIN = 2  # quant.py:16
BITS_MAX = 24  # quant.py:17
SKETCH_TAG = 0x534B  # rsvd.py:16 (_SKETCH_TAG)
DEFAULT_OVERSAMPLE = 10  # rsvd.py:18
SEED_TAG_A = 0xA0  # pipeline.py:34
SEED_TAG_B = 0xB0  # pipeline.py:35
STAGES = ("rsvd", "scaling", "gemm1", "gemm2", "gemm3")  # pipeline.py:37
DEFAULT_D0 = 64  # pipeline.py:47
JACOBI_TOL = 1e-13  # _kernels/_jacobi.py:10
JACOBI_MAX_SWEEPS = 60  # _kernels/_jacobi.py:11


class OracleError(ValueError):
    """Raised for invalid oracle arguments (mirrors the reference's ValueError family)."""


def bit_cap(bits: int) -> int:
    """2^(bits-1) - 1  (quant.py:20-22)."""
    return (1 << (bits - 1)) - 1


def check_bits(bits) -> int:
    """quant.py:25-28."""
    if not isinstance(bits, (int, np.integer)) or not BITS_MIN <= int(bits) <= BITS_MAX:
        raise OracleError(f"bits must be an integer in [{BITS_MIN}, {BITS_MAX}], got {bits}")
    return int(bits)


def as_matrix(a) -> np.ndarray:
    """float64 C-contiguous 2-D coercion (matcore.py:31-38); fp32 upcasts exactly."""
    arr = np.asarray(a, dtype=np.float64)
    if arr.ndim != 2 or arr.shape[0] < 1 or arr.shape[1] < 1:
        raise OracleError(f"expected a non-empty 2-D matrix, got shape {arr.shape}")
    return np.ascontiguousarray(arr)


def rng(seed, *context) -> np.random.Generator:
    """Counter-based generator keyed by seed + context ints (matcore.py:89-92)."""
    entropy = [int(seed) & 0xFFFFFFFFFFFFFFFF] + [int(c) & 0xFFFFFFFFFFFFFFFF for c in context]
    return np.random.Generator(np.random.Philox(np.random.SeedSequence(entropy)))


def child_seeds(seed) -> tuple[int, int]:
    """(seed_A, seed_B) for the two sketches (pipeline.py:152-156)."""
    state = np.random.SeedSequence(
        [int(seed) & 0xFFFFFFFFFFFFFFFF, SEED_TAG_A, SEED_TAG_B]
    ).generate_state(2, dtype=np.uint64)
    return int(state[0]), int(state[1])


def sketch_width(shape, rank: int, oversample: int) -> int:
    """w = min(rank + oversample, min(shape)) (rsvd.py:39-44)."""
    lo = min(shape)
    if rank > lo:
        raise OracleError(f"rank {rank} exceeds min dim {lo} of {shape}")
    return min(rank + oversample, lo)


def gaussian_sketch(seed, ncols: int, width: int) -> np.ndarray:
    """Omega (ncols x width) exactly as rsvd.py:56 draws it."""
    return rng(seed, SKETCH_TAG, ncols, width).standard_normal((ncols, width))


# --------------------------------------------------------------------------
# quantizer (quant.py:55-71 + _core.pyx:53-69 / _pure.py:24-26)


def scale_round_clip(a: np.ndarray, scale, cap: int) -> np.ndarray:
    """rint(a*scale) half-to-even, clamp to +-cap, int32 (_pure.py:24-26).

    ``scale`` may be a scalar or an array broadcastable against ``a`` (per-row /
    per-column restatement: each row / column quantized as its own matrix).
    """
    return np.clip(np.rint(a * scale), -cap, cap).astype(np.int32)


def quantize_tensor(a, bits: int) -> tuple[np.ndarray, float]:
    """Per-tensor symmetric quantizer (quant.py:55-71): returns (int32 data, scale)."""
    a = as_matrix(a)
    bits = check_bits(bits)
    if not np.isfinite(a).all():
        raise OracleError("cannot quantize non-finite entries")
    cap = bit_cap(bits)
    amax = float(np.max(np.abs(a)))
    if amax == 0.0:
        return np.zeros(a.shape, dtype=np.int32), 1.0
    scale = cap / amax
    return scale_round_clip(a, scale, cap), scale


def quantize_rows(a, bits: int) -> tuple[np.ndarray, np.ndarray]:
    """quant.quantize applied to every row as a 1 x n matrix (SURVEY §8(c) CPU restatement).

    Same fp64 ``cap / amax`` per row, same rint / clamp, zero-row sentinel 1.0.
    """
    a = as_matrix(a)
    bits = check_bits(bits)
    if not np.isfinite(a).all():
        raise OracleError("cannot quantize non-finite entries")
    cap = bit_cap(bits)
    amax = np.max(np.abs(a), axis=1)
    scale = np.ones_like(amax)
    nz = amax != 0.0
    scale[nz] = float(cap) / amax[nz]  # IEEE division per element, same as python float
    data = scale_round_clip(a, scale[:, None], cap)
    return data, scale


def quantize_cols(a, bits: int) -> tuple[np.ndarray, np.ndarray]:
    """Per-column quantizer = quantize_rows of the transpose, transposed back."""
    data, scale = quantize_rows(as_matrix(a).T, bits)
    return np.ascontiguousarray(data.T), scale


def quantize(a, bits: int, granularity: str = "tensor"):
    if granularity == "tensor":
        return quantize_tensor(a, bits)
    if granularity == "row":
        return quantize_rows(a, bits)
    if granularity == "col":
        return quantize_cols(a, bits)
    raise OracleError(f"unknown granularity {granularity!r}")


def dequantize(data: np.ndarray, scale) -> np.ndarray:
    """data / scale in float64 (quant.py:74-76)."""
    return data.astype(np.float64) / scale


def check_overflow(k: int, bits_a: int, bits_b: int) -> None:
    """quant.py:87-93: k*cap_a*cap_b must stay below 2^63."""
    if k * bit_cap(bits_a) * bit_cap(bits_b) >= 1 << 63:
        raise OracleError(f"k={k} with bit budgets ({bits_a}, {bits_b}) risks int64 overflow")


def imatmul(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """Exact integer product, int64 result (_core.pyx:35-50 / _pure.py:17-21).

    Accelerated exactly as SURVEY §8(c) prescribes: when every partial sum is
    below 2^53 the float64 BLAS product of the integer operands is exact, and is
    therefore bit-identical to the reference's int64 loop.
    """
    if a.shape[1] != b.shape[0]:
        raise OracleError("inner dimensions differ")
    amax = int(np.max(np.abs(a))) if a.size else 0
    bmax = int(np.max(np.abs(b))) if b.size else 0
    if a.shape[1] * amax * bmax < (1 << 53):
        return (a.astype(np.float64) @ b.astype(np.float64)).astype(np.int64)
    return a.astype(np.int64) @ b.astype(np.int64)


def qgemm(a, b, bits_a: int, bits_b: int, alpha=1.0, beta=0.0, c=None) -> np.ndarray:
    """Per-tensor quantized GEMM (quant.py:96-121)."""
    a = as_matrix(a)
    b = as_matrix(b)
    if a.shape[1] != b.shape[0]:
        raise OracleError(f"inner dimensions differ: {a.shape} @ {b.shape}")
    if c is not None:
        c = as_matrix(c)
    bits_a = check_bits(bits_a)
    bits_b = check_bits(bits_b)
    check_overflow(a.shape[1], bits_a, bits_b)
    qa, sa = quantize_tensor(a, bits_a)
    qb, sb = quantize_tensor(b, bits_b)
    prod = imatmul(qa, qb).astype(np.float64) / (sa * sb)
    if beta != 0.0 and c is not None:
        return alpha * prod + beta * c
    if alpha != 1.0:
        return alpha * prod
    return prod


def qgemm_scaled(a, b, bits_a: int, bits_b: int, granularity: str) -> np.ndarray:
    """Quantized product with per-tensor or per-row(A)/per-column(B) scales.

    granularity "tensor" is exactly `qgemm`; "row" quantizes the rows of A and
    the columns of B independently (each as its own matrix) and dequantizes with
    acc / (sa[:,None] * sb[None,:]), the elementwise analogue of quant.py:116.
    """
    if granularity == "tensor":
        return qgemm(a, b, bits_a, bits_b)
    a = as_matrix(a)
    b = as_matrix(b)
    if a.shape[1] != b.shape[0]:
        raise OracleError(f"inner dimensions differ: {a.shape} @ {b.shape}")
    check_overflow(a.shape[1], bits_a, bits_b)
    qa, sa = quantize_rows(a, bits_a)
    qb, sb = quantize_cols(b, bits_b)
    return imatmul(qa, qb).astype(np.float64) / (sa[:, None] * sb[None, :])


# --------------------------------------------------------------------------
# dense SVD (the `_pure` backend: LAPACK gesdd, _pure.py:29-35)


def svd(a: np.ndarray):
    u, s, vh = np.linalg.svd(a, full_matrices=False)
    return np.ascontiguousarray(u), s, np.ascontiguousarray(vh.T)


def jacobi_svd(a: np.ndarray):
    """Pure-NumPy restatement of the compiled Jacobi oracle (_jacobi.py:14-50 + _core.pyx:72-133).

    Cyclic one-sided Jacobi with per-sweep column-norm refresh, tolerance 1e-13,
    at most 60 sweeps, stable descending sort.  Slow (Python loop over pairs);
    used only on tiny matrices to pin semantics.
    """
    w = np.array(a, dtype=np.float64, order="C", copy=True)
    m, n = w.shape
    transposed = m < n
    if transposed:
        w = np.ascontiguousarray(w.T)
        m, n = n, m
    v = np.eye(n)
    done = -1
    for sweep in range(JACOBI_MAX_SWEEPS):
        colsq = np.einsum("ij,ij->j", w, w)
        worst = 0.0
        rotated = False
        for p in range(n - 1):
            for q in range(p + 1, n):
                app, aqq = colsq[p], colsq[q]
                if app == 0.0 or aqq == 0.0:
                    continue
                apq = float(w[:, p] @ w[:, q])
                if abs(apq) <= JACOBI_TOL * math.sqrt(app * aqq):
                    worst = max(worst, abs(apq) / math.sqrt(app * aqq))
                    continue
                rotated = True
                tau = (aqq - app) / (2.0 * apq)
                t = (1.0 if tau >= 0 else -1.0) / (abs(tau) + math.sqrt(1.0 + tau * tau))
                c = 1.0 / math.sqrt(1.0 + t * t)
                s = c * t
                wp, wq = w[:, p].copy(), w[:, q].copy()
                w[:, p], w[:, q] = c * wp - s * wq, s * wp + c * wq
                vp, vq = v[:, p].copy(), v[:, q].copy()
                v[:, p], v[:, q] = c * vp - s * vq, s * vp + c * vq
                colsq[p] = c * c * app - 2.0 * c * s * apq + s * s * aqq
                colsq[q] = s * s * app + 2.0 * c * s * apq + c * c * aqq
        if not rotated and worst <= JACOBI_TOL:
            done = sweep + 1
            break
    if done < 0:
        raise RuntimeError("jacobi sweeps did not converge")
    sigma = np.sqrt(np.einsum("ij,ij->j", w, w))
    order = np.argsort(-sigma, kind="stable")
    sigma, w, v = sigma[order], w[:, order], v[:, order]
    good = sigma > (sigma[0] * 1e-12 if sigma[0] > 0 else 0.0)
    u = np.zeros_like(w)
    u[:, good] = w[:, good] / sigma[good]
    if not good.all():
        # orthonormal completion (_jacobi.py:53-73)
        basis = [u[:, j] for j in np.nonzero(good)[0]]
        cand = 0
        for j in np.nonzero(~good)[0]:
            while True:
                e = np.zeros(w.shape[0])
                e[cand] = 1.0
                cand += 1
                for _ in range(2):
                    for bvec in basis:
                        e -= (bvec @ e) * bvec
                nrm = math.sqrt(e @ e)
                if nrm > 1e-8:
                    e /= nrm
                    break
            u[:, j] = e
            basis.append(e)
    if transposed:
        u, v = v, u
    return u, sigma, v


# --------------------------------------------------------------------------
# randomized SVD (rsvd.py:47-94) with the fast-mode product extension


@dataclass(frozen=True)
class SketchSpec:
    """How the sketch / power / projection products are evaluated.

    ``None`` bits = fp64 (the reference).  ``granularity`` applies to the
    quantized products: "tensor" (the reference quantizer) or "row" (rows of
    the left operand / columns of the right operand scaled independently).
    """

    sketch_bits: int | None = None
    power_bits: int | None = None
    proj_bits: int | None = None
    granularity: str = "tensor"


def _product(x: np.ndarray, y: np.ndarray, bits: int | None, granularity: str) -> np.ndarray:
    if bits is None:
        return x @ y  # matcore.gemm -> _kernels.matmul (matcore.py:133-152)
    return qgemm_scaled(x, y, bits, bits, granularity)


def range_finder(a, rank: int, power_iters: int, oversample: int, seed, spec=SketchSpec()):
    """Q = orth((A A^T)^q A Omega) with re-orthonormalisation (rsvd.py:47-65)."""
    a = as_matrix(a)
    m, n = a.shape
    width = sketch_width(a.shape, rank, oversample)
    omega = gaussian_sketch(seed, n, width)
    g = spec.granularity
    y = _product(a, omega, spec.sketch_bits, g)
    q = np.linalg.qr(y)[0]
    at = np.ascontiguousarray(a.T)
    for _ in range(power_iters):
        z = _product(at, np.ascontiguousarray(q), spec.power_bits, g)
        qz = np.linalg.qr(z)[0]
        y = _product(a, np.ascontiguousarray(qz), spec.power_bits, g)
        q = np.linalg.qr(y)[0]
    return np.ascontiguousarray(q)


@dataclass(frozen=True)
class Factors:
    u: np.ndarray
    sigma: np.ndarray
    v: np.ndarray


def rsvd(a, rank: int, power_iters: int = 0, oversample: int = DEFAULT_OVERSAMPLE, seed=0,
         spec=SketchSpec(), svd_fn=svd) -> Factors:
    """Randomized thin SVD truncated to ``rank`` (rsvd.py:68-81, truncate rsvd.py:84-94).

    The projection Bs = Q^T A (rsvd.py:77) is evaluated at ``spec.proj_bits``;
    in fast mode it is computed as (A^T Q)^T so the quantized left operand is
    A^T (per-column scales of A) and the right operand is Q.
    """
    a = as_matrix(a)
    q = range_finder(a, rank, power_iters, oversample, seed, spec)
    if spec.proj_bits is None:
        bs = np.ascontiguousarray(q.T) @ a
    else:
        bs = np.ascontiguousarray(
            _product(np.ascontiguousarray(a.T), q, spec.proj_bits, spec.granularity).T
        )
    su, ss, sv = svd_fn(bs)
    u = q @ su
    if rank > ss.shape[0]:
        raise OracleError(f"rank {rank} exceeds factorization width {ss.shape[0]}")
    return Factors(
        u=np.ascontiguousarray(u[:, :rank]),
        sigma=ss[:rank].copy(),
        v=np.ascontiguousarray(sv[:, :rank]),
    )


# --------------------------------------------------------------------------
# the pipeline (pipeline.py:159-214)


@dataclass(frozen=True)
class OracleParams:
    rank: int
    bits: tuple = (8, 8, 4)  # pipeline.py:55
    power_iters: int = 0
    oversample: int = DEFAULT_OVERSAMPLE
    seed: int = 0
    alpha: float = 1.0
    beta: float = 0.0
    spec: SketchSpec = field(default_factory=SketchSpec)


def recombine(fa: Factors, fb: Factors, bits, alpha=1.0, beta=0.0, c=None) -> np.ndarray:
    """Scaling block + three QM products + alpha/beta (pipeline.py:188-210)."""
    d1, d2, d3 = bits
    u_scaled = np.ascontiguousarray(fa.u * fa.sigma)  # m x r
    z_scaled = np.ascontiguousarray((fb.v * fb.sigma).T)  # r x n
    vt = np.ascontiguousarray(fa.v.T)  # r x k
    w = fb.u  # k x r
    e1 = qgemm(vt, w, d1, d1)
    e2 = qgemm(e1, z_scaled, d2, d2)
    e3 = qgemm(u_scaled, e2, d3, d3)
    if beta != 0.0 and c is not None:
        return alpha * e3 + beta * as_matrix(c)
    if alpha != 1.0:
        return alpha * e3
    return e3


def lramm(a, b, params: OracleParams, c=None, svd_fn=svd, return_factors=False):
    """Approximate alpha*A@B + beta*C through the three-stage pipeline (pipeline.py:159-214)."""
    a = as_matrix(a)
    b = as_matrix(b)
    m, k = a.shape
    k2, n = b.shape
    if k != k2:
        raise OracleError(f"inner dimensions differ: {a.shape} @ {b.shape}")
    if params.rank > min(m, k) or params.rank > min(k, n):
        raise OracleError(f"rank {params.rank} exceeds operand min dims")
    seed_a, seed_b = child_seeds(params.seed)
    fa = rsvd(a, params.rank, params.power_iters, params.oversample, seed_a, params.spec, svd_fn)
    fb = rsvd(b, params.rank, params.power_iters, params.oversample, seed_b, params.spec, svd_fn)
    d = recombine(fa, fb, params.bits, params.alpha, params.beta, c)
    if return_factors:
        return d, fa, fb
    return d


def cost_model(m, n, k, r, d0=DEFAULT_D0, d1=8, d2=8, d3=8) -> dict:
    """d^2-weighted MAC model, verbatim formulas of pipeline.py:108-134."""
    d0sq, d1sq, d2sq, d3sq = d0 * d0, d1 * d1, d2 * d2, d3 * d3
    return dict(
        d0=d0,
        rsvd=round(d0sq * ((m + n) * k * math.log2(r) + (m + n + 2 * k) * r * r)),
        scaling=d0sq * (m * r + n * r),
        gemm1=d0sq * 2 * k * r + d2sq * k * r * r,
        gemm2=d0sq * (r * r + n * r) + d3sq * n * r * r,
        gemm3=d0sq * (n * r + m * r) + d1sq * m * n * r,
        baseline_qgemm=d1sq * m * n * k,
        exact_gemm=d0sq * m * n * k,
    )


# --------------------------------------------------------------------------
# synthetic inputs -- shared by tests and bench


def spectrum(kind: str, t: int) -> np.ndarray:
    """i = 1..t: 'exp:tau' -> exp(-i/tau) + 1e-4 ; 'poly:alpha' -> i^-alpha."""
    i = np.arange(1, t + 1, dtype=np.float64)
    name, val = kind.split(":")
    if name == "exp":
        return np.exp(-i / float(val)) + 1e-4
    if name == "poly":
        return i ** (-float(val))
    raise OracleError(f"unknown spectrum {kind!r}")


def synth(rows: int, cols: int, kind: str, cfg: int, idx: int, role: int) -> np.ndarray:
    """A = (U*sigma) @ V^T with Haar U, V; returned as float32 (the device input dtype)."""
    g = np.random.Generator(np.random.Philox(np.random.SeedSequence([0x1A3A, cfg, idx, role])))
    t = min(rows, cols)

    def haar(nr):
        q, r = np.linalg.qr(g.standard_normal((nr, t)))
        return q * np.sign(np.diag(r))

    u = haar(rows)
    v = haar(cols)
    a = (u * spectrum(kind, t)) @ v.T
    return np.ascontiguousarray(a.astype(np.float32))


def generate(rows: int, cols: int, kind: str, seed: int, rank: int = 0, noise_sigma: float = 0.0):
    """Restatement of matcore.generate (matcore.py:95-126) for test inputs."""
    tags = {"uniform": 1, "normal": 2, "exponential": 3, "binary": 4, "lowrank": 5}
    g = rng(seed, tags[kind], rows, cols, rank)
    if kind == "uniform":
        a = g.random((rows, cols))
    elif kind == "normal":
        a = g.standard_normal((rows, cols))
    elif kind == "exponential":
        a = g.standard_exponential((rows, cols))
    elif kind == "binary":
        a = g.integers(0, 2, size=(rows, cols)).astype(np.float64)
    elif kind == "lowrank":
        u = np.linalg.qr(g.standard_normal((rows, rank)))[0]
        v = np.linalg.qr(g.standard_normal((cols, rank)))[0]
        a = (u * (1.0 / np.arange(1, rank + 1))) @ v.T
        if noise_sigma > 0:
            a = a + noise_sigma * g.standard_normal((rows, cols))
    else:
        raise OracleError(f"unknown kind {kind!r}")
    return np.ascontiguousarray(a)


def rel_fro(x, ref) -> float:
    x = np.asarray(x, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    den = float(np.linalg.norm(ref))
    num = float(np.linalg.norm(x - ref))
    return num / den if den > 0 else num
