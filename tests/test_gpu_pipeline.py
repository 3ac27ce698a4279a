"""End-to-end parity of the device pipeline against the oracle / reference goldens.

Gates:
  L2  recombination: given the same factors, E1 -> E2 -> E3 is bit-identical.
  L3  factorisation: sigma to 1e-10 relative, sign-invariant subspaces to 1e-9.
  L4  parity mode end to end: <= 1e-9 relative Frobenius vs the reference's lramm()
      (the reference's own two kernel backends differ by up to ~2e-3 on rare seeds:
      the chained per-tensor quantisers are discontinuous).
  L5  fast mode (int8 sketches): <= 1e-3 vs the CPU restatement at the same seeds,
      and error vs the exact product within 2 % of the reference's.
"""

import os
import sys

import numpy as np
import pytest

import lramm_oracle as O

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

HERE = os.path.dirname(os.path.abspath(__file__))
G = np.load(os.path.join(HERE, "golden", "reference_golden.npz"))
sys.path.insert(0, os.path.join(HERE, "golden"))
import cases as MG  # noqa: E402  (case tables only; does not import the reference)


@pytest.fixture(scope="module")
def L():
    import paper_2405_16917_b200 as lib

    return lib


def subspace_err(x, y):
    """|| X X^T - Y Y^T ||_F for orthonormal-column X, Y (sign/rotation invariant)."""
    return np.linalg.norm(x @ x.T - y @ y.T)


# ------------------------------------------------------------------ L2 recombination


@pytest.mark.parametrize("bits", [(8, 8, 8), (8, 8, 4), (8, 4, 8), (4, 4, 4)])
def test_recombination_bitwise_given_factors(L, bits):
    a = O.synth(200, 150, "exp:10", 4, 0, 0)
    b = O.synth(150, 170, "exp:10", 4, 0, 1)
    _, fa, fb = O.lramm(a, b, O.OracleParams(rank=20, bits=bits, power_iters=1, oversample=8), return_factors=True)
    ref = O.recombine(fa, fb, bits)
    d1, d2, d3 = bits
    e1 = L.qgemm(np.ascontiguousarray(fa.v.T), fb.u, d1, d1)
    e2 = L.qgemm(e1, np.ascontiguousarray((fb.v * fb.sigma).T), d2, d2)
    e3 = L.qgemm(np.ascontiguousarray(fa.u * fa.sigma), e2, d3, d3)
    assert np.array_equal(e3, ref)


# ------------------------------------------------------------------ L3 rsvd


@pytest.mark.parametrize("name", ["rs_a", "rs_b"])
def test_rsvd_matches_reference_golden(L, name):
    rows, cols, kind, rank, q_iters, p, seed = {
        "rs_a": (90, 70, "exp:6", 10, 1, 5, 11),
        "rs_b": (60, 100, "poly:1.2", 12, 0, 10, 12),
    }[name]
    x = O.synth(rows, cols, kind, 2, seed, 0)
    f = L.rsvd(x, L.RsvdParams(rank, q_iters, p, seed))
    s_ref = G[name + "_s"]
    assert np.max(np.abs(f.sigma - s_ref)) <= 1e-10 * s_ref[0]
    assert subspace_err(f.u, G[name + "_u"]) <= 1e-9
    assert subspace_err(f.v, G[name + "_v"]) <= 1e-9
    assert np.linalg.norm(f.u.T @ f.u - np.eye(rank)) <= 1e-8 * np.sqrt(rank)


def test_rsvd_exact_rank_one(L):
    # test_rsvd.py:68-76: rank-deficient sketch -> Householder fallback on device
    u = np.zeros((30, 1))
    u[4, 0] = 1.0
    v = np.zeros((20, 1))
    v[11, 0] = 1.0
    a = 3.0 * u @ v.T
    f = L.rsvd(a, L.RsvdParams(rank=1, seed=5))
    assert abs(float(f.sigma[0]) - 3.0) <= 1e-8
    assert np.linalg.norm(a - (f.u * f.sigma) @ f.v.T) <= 1e-8


@pytest.mark.parametrize("spectrum", ["exp:24", "poly:1.5", "poly:3"])
def test_rsvd_fast_mode_matches_restatement(L, spectrum):
    # exp:24 keeps every sketch well conditioned (single CholeskyQR pass in fast mode); the
    # polynomial spectra push kappa(Y) past the second-pass threshold
    x = O.synth(512, 384, spectrum, 6, 0, 0)
    for gran in ("tensor", "row"):
        spec = O.SketchSpec(8, 8, 8, gran)
        f_ref = O.rsvd(x, 32, 1, 8, 123, spec)
        f = L.rsvd(x, L.RsvdParams(32, 1, 8, 123, mode="fast", sketch_bits=8, power_bits=8, proj_bits=8,
                                   granularity=gran))
        assert np.max(np.abs(f.sigma - f_ref.sigma)) <= 1e-9 * f_ref.sigma[0]
        assert subspace_err(f.u[:, :16], f_ref.u[:, :16]) <= 1e-8


def test_range_finder_contracts(L):
    q = L.range_finder(np.eye(4), L.RsvdParams(rank=2, oversample=0, seed=1))  # test_rsvd.py:34-37
    assert q.shape == (4, 2) and np.linalg.norm(q.T @ q - np.eye(2)) <= 1e-8
    a = O.generate(60, 50, "lowrank", 2, rank=3)
    q = L.range_finder(a, L.RsvdParams(rank=3, oversample=2, seed=3))
    assert np.linalg.norm(a - q @ (q.T @ a)) <= 1e-8 * np.linalg.norm(a)
    q = L.range_finder(np.eye(6), L.RsvdParams(rank=4, oversample=50, seed=1))
    assert q.shape == (6, 6)


# ------------------------------------------------------------------ L4 parity mode


@pytest.mark.parametrize("idx", range(len(MG.LRAMM_CASES)))
def test_lramm_parity_vs_reference_golden(L, idx):
    name, m, k, n, kind, rank, p, q_iters, bits, seed = MG.LRAMM_CASES[idx]
    a = O.synth(m, k, kind, 3, seed, 0)
    b = O.synth(k, n, kind, 3, seed, 1)
    d, timings = L.lramm(a, b, L.LrammParams(rank=rank, bits=bits, power_iters=q_iters, oversample=p, seed=seed))
    assert d.dtype == np.float64 and d.shape == (m, n)
    ref = G[f"lr_{name}_pure"]
    # the reference's two kernel backends agree to <= 2.2e-13 on every one of these cases, so
    # the gate is the SURVEY §8(c) L4 bound, 1e-9 (not the BASELINE 1e-3 target)
    assert O.rel_fro(G[f"lr_{name}_compiled"], ref) <= 1e-12
    assert O.rel_fro(d, ref) <= 1e-9
    assert set(timings.wall_ns) == set(L.STAGES)


@pytest.mark.parametrize("idx", range(len(MG.LOWRANK_CASES)))
def test_lramm_lowrank_inputs(L, idx):
    name, m, k, n, lr_rank, rank, p, q_iters, bits, seed = MG.LOWRANK_CASES[idx]
    a = O.generate(m, k, "lowrank", seed, rank=lr_rank)
    b = O.generate(k, n, "lowrank", seed + 100, rank=lr_rank)
    d, _ = L.lramm(a, b, L.LrammParams(rank=rank, bits=bits, power_iters=q_iters, oversample=p, seed=seed))
    exact = a @ b
    spread = O.rel_fro(G[f"lr_{name}_compiled"], G[f"lr_{name}_pure"])
    if spread <= 1e-12:  # the reference's backends agree: the L4 gate
        assert O.rel_fro(d, G[f"lr_{name}_pure"]) <= 1e-9
        return
    # rank-deficient operands (rank < params.rank): the trailing singular triplets are an
    # arbitrary orthonormal completion in the reference too (its LAPACK and Jacobi backends
    # pick different ones), and they enter E1's per-tensor scale.  Gate: accuracy vs the exact
    # product within the spread of the reference's own two backends.
    errs = [O.rel_fro(G[f"lr_{name}_{k}"], exact) for k in ("pure", "compiled")]
    assert O.rel_fro(d, exact) <= 2.0 * max(errs) + 0.02


def test_lramm_config1_parity(L):
    a = O.synth(1024, 1024, "exp:32", 1, 0, 0)
    b = O.synth(1024, 1024, "exp:32", 1, 0, 1)
    d, _ = L.lramm(a, b, L.LrammParams(rank=64, bits=(8, 8, 8), power_iters=1, oversample=10, seed=0))
    assert abs(np.linalg.norm(d) - float(G["c1_fro"])) <= 1e-9 * float(G["c1_fro"])
    assert O.rel_fro(d.sum(axis=1), G["c1_rowsum"]) <= 1e-9
    assert O.rel_fro(d.sum(axis=0), G["c1_colsum"]) <= 1e-9
    assert O.rel_fro(d[:32, :32], G["c1_block"]) <= 1e-9
    exact = a.astype(np.float64) @ b.astype(np.float64)
    assert abs(O.rel_fro(d, exact) - float(G["c1_relerr_exact"])) <= 0.02 * float(G["c1_relerr_exact"])


def test_lramm_alpha_beta_and_c_independence(L):
    a = O.generate(40, 30, "uniform", 11)
    b = O.generate(30, 50, "uniform", 12)
    c = O.generate(40, 50, "normal", 13)
    base, _ = L.lramm(a, b, L.LrammParams(rank=4, seed=14))
    same, _ = L.lramm(a, b, L.LrammParams(rank=4, seed=14), c=c)  # beta defaults to 0
    assert np.array_equal(base, same)
    combo, _ = L.lramm(a, b, L.LrammParams(rank=4, seed=14, alpha=2.0, beta=-1.0), c=c)
    ref = O.lramm(a, b, O.OracleParams(rank=4, seed=14, alpha=2.0, beta=-1.0), c=c)
    assert np.allclose(combo, 2.0 * base - c, atol=1e-12)
    assert O.rel_fro(combo, ref) <= 1e-3


def test_lramm_deterministic_bitwise(L):
    a = O.generate(130, 130, "normal", 15)
    b = O.generate(130, 130, "normal", 16)
    params = L.LrammParams(rank=5, bits=(8, 8, 4), seed=17)
    d1, _ = L.lramm(a, b, params)
    d2, _ = L.lramm(a, b, params)
    assert np.array_equal(d1, d2)


def test_lramm_device_tensors_and_fp32_output(L):
    a = O.synth(256, 192, "exp:16", 1, 0, 0)
    b = O.synth(192, 224, "exp:16", 1, 0, 1)
    params = L.LrammParams(rank=24, bits=(8, 8, 8), power_iters=1, oversample=6, seed=3)
    d_host, _ = L.lramm(a, b, params)
    ta = torch.from_numpy(a).cuda()
    tb = torch.from_numpy(b).cuda()
    d_dev, _ = L.lramm(ta, tb, params)
    assert np.array_equal(d_dev.cpu().numpy(), d_host)
    p32 = L.LrammParams(rank=24, bits=(8, 8, 8), power_iters=1, oversample=6, seed=3, out_dtype=np.float32)
    d32, _ = L.lramm(a, b, p32)
    assert d32.dtype == np.float32 and np.array_equal(d32, d_host.astype(np.float32))


@pytest.mark.parametrize("bits", [(16, 16, 16), (24, 12, 8), (8, 8, 16)])
def test_lramm_high_bit_budgets(L, bits):
    """Bit budgets 9..24 in the recombination (test_pipeline.py:28-41 uses 16/24): limb products."""
    a = O.synth(200, 160, "exp:12", 3, 0, 0)
    b = O.synth(160, 180, "exp:12", 3, 0, 1)
    kw = dict(rank=12, bits=bits, power_iters=1, oversample=6, seed=9)
    d, _ = L.lramm(a, b, L.LrammParams(**kw))
    ref = O.lramm(a, b, O.OracleParams(**kw))
    ref2 = O.lramm(a, b, O.OracleParams(**kw), svd_fn=O.jacobi_svd)
    assert min(O.rel_fro(d, ref), O.rel_fro(d, ref2)) <= max(1e-3, 1.5 * O.rel_fro(ref2, ref))
    # and the recombination itself is bit-exact given the same factors (L2 gate, limb products)
    fa = O.rsvd(a, 12, 1, 6, O.child_seeds(9)[0])
    fb = O.rsvd(b, 12, 1, 6, O.child_seeds(9)[1])
    e = O.recombine(fa, fb, bits)
    e1 = L.qgemm(np.ascontiguousarray(fa.v.T), fb.u, bits[0], bits[0])
    e2 = L.qgemm(e1, np.ascontiguousarray((fb.v * fb.sigma).T), bits[1], bits[1])
    e3 = L.qgemm(np.ascontiguousarray(fa.u * fa.sigma), e2, bits[2], bits[2])
    assert np.array_equal(e3, e)


def test_lramm_nonfinite_input_raises(L):
    a = np.ones((20, 20))
    a[3, 4] = np.nan
    with pytest.raises((L.ParameterError, RuntimeError)):
        L.lramm(a, np.eye(20), L.LrammParams(rank=4))


# ------------------------------------------------------------------ L5 fast mode


@pytest.mark.parametrize("shape", [(512, 384, 448), (300, 257, 199), (96, 33, 80)])
@pytest.mark.parametrize("gran", ["tensor", "row"])
def test_lramm_int4_sketch_vs_restatement(L, gran, shape):
    # 4-bit sketch budget: X travels as packed int4 and is unpacked to int8 in shared memory by the
    # GEMM (c3's Y = A . Omega); odd K exercises the half-filled last byte of each packed row
    m, k, n = shape
    a = O.synth(m, k, "exp:24", 9, 0, 0)
    b = O.synth(k, n, "exp:24", 9, 0, 1)
    kw = dict(rank=16, bits=(8, 8, 8), power_iters=1, oversample=6, seed=3)
    ref = O.lramm(a, b, O.OracleParams(**kw, spec=O.SketchSpec(4, 8, 8, gran)))
    d, _ = L.lramm(a, b, L.LrammParams(**kw, mode="fast", sketch_bits=4, power_bits=8, proj_bits=8, granularity=gran))
    assert O.rel_fro(d, ref) <= 1e-3
    f_ref = O.rsvd(a, 16, 1, 6, 7, O.SketchSpec(4, 4, 8, gran))  # power iteration at 4 bits too (packed X twice)
    f = L.rsvd(a, L.RsvdParams(16, 1, 6, 7, mode="fast", sketch_bits=4, power_bits=4, proj_bits=8, granularity=gran))
    assert np.max(np.abs(f.sigma - f_ref.sigma)) <= 1e-9 * f_ref.sigma[0]


@pytest.mark.parametrize("gran", ["tensor", "row"])
def test_lramm_fast_mode_vs_restatement(L, gran):
    a = O.synth(512, 512, "exp:24", 7, 0, 0)
    b = O.synth(512, 512, "exp:24", 7, 0, 1)
    exact = a.astype(np.float64) @ b.astype(np.float64)
    kw = dict(rank=32, bits=(8, 8, 8), power_iters=1, oversample=8, seed=5)
    spec = O.SketchSpec(8, 8, 8, gran)
    ref = O.lramm(a, b, O.OracleParams(**kw, spec=spec))
    d, _ = L.lramm(a, b, L.LrammParams(**kw, mode="fast", sketch_bits=8, power_bits=8, proj_bits=8, granularity=gran))
    assert O.rel_fro(d, ref) <= 1e-3
    e_ref_par = O.rel_fro(O.lramm(a, b, O.OracleParams(**kw)), exact)
    assert abs(O.rel_fro(d, exact) - e_ref_par) <= 0.02 * e_ref_par
