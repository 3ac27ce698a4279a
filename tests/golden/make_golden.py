"""Generate golden vectors by running the UNMODIFIED reference (test infrastructure).

Run in the build container, where the reference is installed into `oracle/_ref`
by `oracle/build_ref.sh`:

    PYTHONPATH=oracle/_ref python tests/golden/make_golden.py

Writes `tests/golden/reference_golden.npz`.  Every array in it is an output of
the reference's own public API (`lramm.quantize`, `lramm.qgemm`,
`lramm.integer_matmul`, `lramm.rsvd`, `lramm.lramm`, `lramm._kernels`), called on
seeded inputs that the tests regenerate bit-identically with NumPy's Philox.
`lramm()` goldens are produced with the reference's "python" kernel backend
(`LRAMM_PURE_PYTHON` semantics, `_kernels/_pure.py`) *and* its compiled Cython
backend; both are stored so tests can show the reference's own backend spread.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle", "_ref"))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, HERE)

import lramm  # noqa: E402  (the reference)
import lramm._kernels as K  # noqa: E402
from lramm._kernels import _pure  # noqa: E402

import lramm_oracle as O  # noqa: E402  (only for the shared seeded input generators)


def _pure_backend():
    class _Ctx:
        def __enter__(self):
            self.saved = (K.matmul, K.imatmul, K.scale_round_clip, K.svd)
            K.matmul, K.imatmul, K.scale_round_clip, K.svd = (
                _pure.matmul, _pure.imatmul, _pure.scale_round_clip, _pure.svd)

        def __exit__(self, *exc):
            K.matmul, K.imatmul, K.scale_round_clip, K.svd = self.saved

    return _Ctx()


from cases import LOWRANK_CASES, LRAMM_CASES  # noqa: E402,F401  (the case tables)


def main():
    out = {}
    # ---- quantize: reference KATs + seeded inputs, bits 2..24 --------------------
    kat = {
        "kat_ext": (np.array([[1.0, -1.0]]), 8),  # test_quant.py:32-35
        "kat_formula": (np.array([[2.0, 0.0]]), 4),  # test_quant.py:38-41
        "kat_zero": (np.zeros((2, 2)), 8),  # test_quant.py:44-47
    }
    for name, (x, bits) in kat.items():
        q = lramm.quantize(x, bits)
        out[f"q_{name}_x"] = x
        out[f"q_{name}_data"] = q.data
        out[f"q_{name}_scale"] = np.float64(q.scale)
        out[f"q_{name}_bits"] = np.int64(bits)
    halves = np.array([[0.5, 1.5, 2.5, -0.5, -1.5, -2.5]])  # test_backends.py:46-51
    out["src_halves_x"] = halves
    out["src_halves_out"] = K.scale_round_clip(halves, 1.0, 127)
    for bits in (2, 3, 4, 5, 8, 12, 16, 24):
        x = O.generate(33, 47, "normal", 100 + bits)
        q = lramm.quantize(x, bits)
        out[f"q_normal_{bits}_data"] = q.data
        out[f"q_normal_{bits}_scale"] = np.float64(q.scale)
    # fp32-valued input (device input dtype), upcast exactly by the reference
    x32 = O.synth(64, 96, "exp:8", 9, 0, 0)
    out["q_fp32_x"] = x32
    q = lramm.quantize(x32, 8)
    out["q_fp32_data"], out["q_fp32_scale"] = q.data, np.float64(q.scale)

    # ---- integer_matmul / qgemm -------------------------------------------------
    a = O.generate(8, 8, "normal", 71)
    b = O.generate(8, 8, "normal", 72)
    out["imm_out"] = lramm.integer_matmul(lramm.quantize(a, 8), lramm.quantize(b, 8))
    for (bits_a, bits_b) in ((8, 8), (4, 8), (6, 6), (2, 3)):
        a = O.generate(21, 35, "uniform", 80 + bits_a)
        b = O.generate(35, 17, "normal", 90 + bits_b)
        out[f"qg_{bits_a}_{bits_b}"] = lramm.qgemm(a, b, bits_a, bits_b)
    a = O.generate(6, 5, "uniform", 83)
    b = O.generate(5, 7, "uniform", 84)
    c = O.generate(6, 7, "normal", 85)
    out["qg_ab"] = lramm.qgemm(a, b, 8, 8, alpha=2.0, beta=3.0, c=c)

    # ---- Jacobi SVD (compiled) -------------------------------------------------
    from lramm._kernels import _jacobi
    for shape in ((20, 20), (35, 14), (14, 35)):
        x = O.generate(*shape, "normal", 5)
        u, s, v = _jacobi.jacobi_svd(x)
        key = f"jac_{shape[0]}x{shape[1]}"
        out[key + "_u"], out[key + "_s"], out[key + "_v"] = u, s, v

    # ---- rsvd factors ------------------------------------------------------------
    for name, (rows, cols, kind, rank, q_iters, p, seed) in {
        "rs_a": (90, 70, "exp:6", 10, 1, 5, 11),
        "rs_b": (60, 100, "poly:1.2", 12, 0, 10, 12),
    }.items():
        x = O.synth(rows, cols, kind, 2, seed, 0).astype(np.float64)
        with _pure_backend():
            f = lramm.rsvd(x, lramm.RsvdParams(rank, q_iters, p, seed))
        out[name + "_u"], out[name + "_s"], out[name + "_v"] = f.u, f.sigma, f.v

    # ---- lramm -------------------------------------------------------------------
    for (name, m, k, n, kind, rank, p, q_iters, bits, seed) in LRAMM_CASES:
        a = O.synth(m, k, kind, 3, seed, 0).astype(np.float64)
        b = O.synth(k, n, kind, 3, seed, 1).astype(np.float64)
        params = lramm.LrammParams(rank=rank, bits=bits, power_iters=q_iters, oversample=p, seed=seed)
        with _pure_backend():
            d_pure, _ = lramm.lramm(a, b, params)
        d_comp, _ = lramm.lramm(a, b, params)
        out[f"lr_{name}_pure"] = d_pure
        out[f"lr_{name}_compiled"] = d_comp
    for (name, m, k, n, lr_rank, rank, p, q_iters, bits, seed) in LOWRANK_CASES:
        a = O.generate(m, k, "lowrank", seed, rank=lr_rank)
        b = O.generate(k, n, "lowrank", seed + 100, rank=lr_rank)
        params = lramm.LrammParams(rank=rank, bits=bits, power_iters=q_iters, oversample=p, seed=seed)
        with _pure_backend():
            d_pure, _ = lramm.lramm(a, b, params)
        d_comp, _ = lramm.lramm(a, b, params)
        out[f"lr_{name}_pure"] = d_pure
        out[f"lr_{name}_compiled"] = d_comp

    # ---- config 1 (BASELINE configs[0]) summary: too large to store whole --------
    a = O.synth(1024, 1024, "exp:32", 1, 0, 0)
    b = O.synth(1024, 1024, "exp:32", 1, 0, 1)
    params = lramm.LrammParams(rank=64, bits=(8, 8, 8), power_iters=1, oversample=10, seed=0)
    with _pure_backend():
        d, _ = lramm.lramm(a, b, params)
    out["c1_rowsum"] = d.sum(axis=1)
    out["c1_colsum"] = d.sum(axis=0)
    out["c1_block"] = d[:32, :32].copy()
    out["c1_fro"] = np.float64(np.linalg.norm(d))
    out["c1_relerr_exact"] = np.float64(
        np.linalg.norm(d - a.astype(np.float64) @ b.astype(np.float64))
        / np.linalg.norm(a.astype(np.float64) @ b.astype(np.float64)))
    out["meta_numpy"] = np.array(np.__version__)
    out["meta_reference"] = np.array(f"lramm {lramm.__version__} ({lramm.backend_name()} core built)")
    path = os.path.join(HERE, "reference_golden.npz")
    np.savez_compressed(path, **out)
    print("wrote", path, os.path.getsize(path), "bytes,", len(out), "arrays")


if __name__ == "__main__":
    main()
