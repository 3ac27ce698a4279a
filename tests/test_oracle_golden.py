"""Pin the CPU oracle (oracle/lramm_oracle.py) against the reference.

Golden vectors in tests/golden/reference_golden.npz were produced by the
unmodified reference (tests/golden/make_golden.py); the known-answer tests are
the reference's own (pkg/tests/test_quant.py, test_backends.py).
"""

import os

import numpy as np
import pytest

import lramm_oracle as O

G = np.load(os.path.join(os.path.dirname(__file__), "golden", "reference_golden.npz"))


def test_quantize_kats():
    # test_quant.py:32-35 / :38-41 / :44-47
    d, s = O.quantize_tensor(np.array([[1.0, -1.0]]), 8)
    assert s == 127.0 and d.tolist() == [[127, -127]]
    d, s = O.quantize_tensor(np.array([[2.0, 0.0]]), 4)
    assert s == 3.5 and d.tolist() == [[7, 0]]
    d, s = O.quantize_tensor(np.zeros((2, 2)), 8)
    assert s == 1.0 and not d.any()
    # test_backends.py:46-51 half-to-even
    out = O.scale_round_clip(G["src_halves_x"], 1.0, 127)
    assert np.array_equal(out, G["src_halves_out"])
    assert out.tolist() == [[0, 2, 2, 0, -2, -2]]


@pytest.mark.parametrize("name", ["kat_ext", "kat_formula", "kat_zero"])
def test_quantize_golden_kat(name):
    d, s = O.quantize_tensor(G[f"q_{name}_x"], int(G[f"q_{name}_bits"]))
    assert np.array_equal(d, G[f"q_{name}_data"])
    assert s == float(G[f"q_{name}_scale"])


@pytest.mark.parametrize("bits", [2, 3, 4, 5, 8, 12, 16, 24])
def test_quantize_golden_bits(bits):
    x = O.generate(33, 47, "normal", 100 + bits)
    d, s = O.quantize_tensor(x, bits)
    assert np.array_equal(d, G[f"q_normal_{bits}_data"])
    assert s == float(G[f"q_normal_{bits}_scale"])


def test_quantize_golden_fp32_input():
    d, s = O.quantize_tensor(G["q_fp32_x"], 8)
    assert np.array_equal(d, G["q_fp32_data"]) and s == float(G["q_fp32_scale"])


def test_rowwise_is_per_row_reference_quantizer():
    x = O.generate(9, 13, "normal", 3)
    x[4] = 0.0
    d, s = O.quantize_rows(x, 6)
    for i in range(x.shape[0]):
        di, si = O.quantize_tensor(x[i : i + 1], 6)
        assert np.array_equal(d[i : i + 1], di) and s[i] == si
    dc, sc = O.quantize_cols(x, 6)
    assert np.array_equal(dc, O.quantize_rows(x.T, 6)[0].T)


def test_integer_matmul_golden():
    a = O.generate(8, 8, "normal", 71)
    b = O.generate(8, 8, "normal", 72)
    out = O.imatmul(O.quantize_tensor(a, 8)[0], O.quantize_tensor(b, 8)[0])
    assert out.dtype == np.int64 and np.array_equal(out, G["imm_out"])


@pytest.mark.parametrize("bits", [(8, 8), (4, 8), (6, 6), (2, 3)])
def test_qgemm_golden(bits):
    a = O.generate(21, 35, "uniform", 80 + bits[0])
    b = O.generate(35, 17, "normal", 90 + bits[1])
    assert np.array_equal(O.qgemm(a, b, *bits), G[f"qg_{bits[0]}_{bits[1]}"])


def test_qgemm_alpha_beta_golden():
    a = O.generate(6, 5, "uniform", 83)
    b = O.generate(5, 7, "uniform", 84)
    c = O.generate(6, 7, "normal", 85)
    assert np.array_equal(O.qgemm(a, b, 8, 8, 2.0, 3.0, c), G["qg_ab"])


@pytest.mark.parametrize("shape", [(20, 20), (35, 14), (14, 35)])
def test_jacobi_restatement_golden(shape):
    x = O.generate(*shape, "normal", 5)
    u, s, v = O.jacobi_svd(x)
    key = f"jac_{shape[0]}x{shape[1]}"
    assert np.max(np.abs(s - G[key + "_s"])) <= 1e-13 * s[0]
    # sign-invariant: the singular triplets agree up to paired signs
    sign = np.sign(np.sum(u * G[key + "_u"], axis=0))
    assert np.max(np.abs(u * sign - G[key + "_u"])) <= 1e-10
    assert np.max(np.abs(v * sign - G[key + "_v"])) <= 1e-10


@pytest.mark.parametrize("name", ["rs_a", "rs_b"])
def test_rsvd_golden(name):
    rows, cols, kind, rank, q_iters, p, seed = {
        "rs_a": (90, 70, "exp:6", 10, 1, 5, 11),
        "rs_b": (60, 100, "poly:1.2", 12, 0, 10, 12),
    }[name]
    x = O.synth(rows, cols, kind, 2, seed, 0)
    f = O.rsvd(x, rank, q_iters, p, seed)
    assert np.array_equal(f.sigma, G[name + "_s"])
    assert np.array_equal(f.u, G[name + "_u"]) and np.array_equal(f.v, G[name + "_v"])




def _load_mg():
    import sys

    sys.path.insert(0, os.path.join(os.path.dirname(__file__), "golden"))
    import cases as MG  # noqa: F401  (only the case tables are used)

    return MG


@pytest.mark.parametrize("idx", range(8))
def test_lramm_golden_parity_mode(idx):
    MG = _load_mg()
    name, m, k, n, kind, rank, p, q_iters, bits, seed = MG.LRAMM_CASES[idx]
    a = O.synth(m, k, kind, 3, seed, 0)
    b = O.synth(k, n, kind, 3, seed, 1)
    d = O.lramm(a, b, O.OracleParams(rank=rank, bits=bits, power_iters=q_iters, oversample=p, seed=seed))
    ref = G[f"lr_{name}_pure"]
    # bitwise on this host (same OpenBLAS); 1e-12 elsewhere
    assert O.rel_fro(d, ref) <= 1e-12
    # the reference's own compiled backend: same algorithm, different summation order
    assert O.rel_fro(G[f"lr_{name}_compiled"], ref) <= 5e-3


@pytest.mark.parametrize("idx", range(2))
def test_lramm_golden_lowrank(idx):
    MG = _load_mg()
    name, m, k, n, lr_rank, rank, p, q_iters, bits, seed = MG.LOWRANK_CASES[idx]
    a = O.generate(m, k, "lowrank", seed, rank=lr_rank)
    b = O.generate(k, n, "lowrank", seed + 100, rank=lr_rank)
    d = O.lramm(a, b, O.OracleParams(rank=rank, bits=bits, power_iters=q_iters, oversample=p, seed=seed))
    assert O.rel_fro(d, G[f"lr_{name}_pure"]) <= 1e-12


def test_lramm_golden_config1():
    a = O.synth(1024, 1024, "exp:32", 1, 0, 0)
    b = O.synth(1024, 1024, "exp:32", 1, 0, 1)
    d = O.lramm(a, b, O.OracleParams(rank=64, bits=(8, 8, 8), power_iters=1, oversample=10, seed=0))
    assert abs(np.linalg.norm(d) - float(G["c1_fro"])) <= 1e-12 * float(G["c1_fro"])
    assert O.rel_fro(d.sum(axis=1), G["c1_rowsum"]) <= 1e-12
    assert O.rel_fro(d.sum(axis=0), G["c1_colsum"]) <= 1e-12
    assert O.rel_fro(d[:32, :32], G["c1_block"]) <= 1e-12


def test_cost_model_matches_reference_formula():
    # README / pipeline.py:108-134: 8192x8192x1024, r=50, d=16, d0=64 -> ~12.13x
    cm = O.cost_model(8192, 8192, 1024, 50, 64, 16, 16, 16)
    total = sum(cm[s] for s in O.STAGES)
    assert abs(cm["baseline_qgemm"] / total - 12.13) < 0.01


def test_fast_mode_restatement_accuracy_parity():
    """Fast mode (int8 per-row sketches) keeps the reference's accuracy vs exact."""
    a = O.synth(256, 256, "exp:16", 9, 0, 0)
    b = O.synth(256, 256, "exp:16", 9, 0, 1)
    exact = a.astype(np.float64) @ b.astype(np.float64)
    par = O.OracleParams(rank=24, bits=(8, 8, 8), power_iters=1, oversample=8, seed=0)
    fast = O.OracleParams(rank=24, bits=(8, 8, 8), power_iters=1, oversample=8, seed=0,
                          spec=O.SketchSpec(8, 8, 8, "row"))
    e_par = O.rel_fro(O.lramm(a, b, par), exact)
    e_fast = O.rel_fro(O.lramm(a, b, fast), exact)
    assert abs(e_fast - e_par) <= 0.02 * e_par
