"""The reference's own behavioural tests for the hot path, run against the B200 package.

Each test restates an assertion of `pkg/tests/test_pipeline.py`, `test_rsvd.py` or
`test_quant.py` (file:line in the docstrings) through `paper_2405_16917_b200` -- the same
inputs (the reference's generators, restated in the oracle), the same thresholds -- so the
drop-in keeps the behaviour the reference promises, including bit budgets up to 24.
"""

import math

import numpy as np
import pytest

import lramm_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def L():
    import paper_2405_16917_b200 as pkg

    return pkg


def gen(rows, cols, kind, seed, rank=0, noise=0.0):
    return O.generate(rows, cols, kind, seed, rank, noise)


def rel(x, ref):
    return float(np.linalg.norm(x - ref) / np.linalg.norm(ref))


# ------------------------------------------------------------------ pipeline (test_pipeline.py)


def test_exact_low_rank_with_wide_budgets(L):
    """test_pipeline.py:28-32"""
    a, b = gen(150, 150, "lowrank", 1, 1), gen(150, 150, "lowrank", 2, 1)
    d, _ = L.lramm(a, b, L.LrammParams(rank=2, bits=(24, 24, 24), seed=3))
    assert rel(d, a @ b) <= 1e-4


def test_full_effective_rank_wide_budgets(L):
    """test_pipeline.py:35-40"""
    a, b = gen(40, 40, "lowrank", 4, 6), gen(40, 40, "lowrank", 5, 6)
    d, _ = L.lramm(a, b, L.LrammParams(rank=6, bits=(24, 24, 24), seed=6))
    assert rel(d, a @ b) <= 1e-3


def test_error_monotone_in_bits(L):
    """test_pipeline.py:88-99"""
    e_high, e_low = [], []
    for seed in range(10):
        a, b = gen(64, 64, "uniform", 1100 + seed), gen(64, 64, "uniform", 1200 + seed)
        d8, _ = L.lramm(a, b, L.LrammParams(rank=8, bits=(8, 8, 8), seed=seed))
        d4, _ = L.lramm(a, b, L.LrammParams(rank=8, bits=(4, 4, 4), seed=seed))
        e_high.append(rel(d8, a @ b))
        e_low.append(rel(d4, a @ b))
    assert np.median(e_high) <= np.median(e_low)


@pytest.mark.parametrize("kind", ["uniform", "lowrank"])
def test_combined_bound_holds(L, kind):
    """test_pipeline.py:102-111"""
    from paper_2405_16917_b200.report import combined_bound

    for seed in range(5):
        a = gen(64, 64, kind, 1300 + seed, 10, 1e-3)
        b = gen(64, 64, kind, 1400 + seed, 10, 1e-3)
        params = L.LrammParams(rank=8, bits=(8, 8, 4), seed=seed)
        d, _ = L.lramm(a, b, params)
        bound, source = combined_bound(a, b, params)
        assert source == "oracle"
        assert np.linalg.norm(d - a @ b) <= bound


def test_lowrank_competitive_with_direct_4bit(L):
    """test_pipeline.py:114-128"""
    e_lr, e_dq4 = [], []
    for seed in range(10):
        a = gen(128, 128, "lowrank", 2 * seed, 10, 1e-3)
        b = gen(128, 128, "lowrank", 2 * seed + 1, 10, 1e-3)
        d, _ = L.lramm(a, b, L.LrammParams(rank=13, bits=(8, 8, 4), seed=seed))
        e_lr.append(rel(d, a @ b))
        e_dq4.append(rel(L.qgemm(a, b, 4, 4), a @ b))
    assert np.median(e_lr) <= 1.2 * np.median(e_dq4)


def test_normal_inputs_favor_direct_quantization(L):
    """test_pipeline.py:131-141"""
    e_lr, e_dq4 = [], []
    for seed in range(10):
        a, b = gen(128, 128, "normal", 2 * seed), gen(128, 128, "normal", 2 * seed + 1)
        d, _ = L.lramm(a, b, L.LrammParams(rank=13, bits=(8, 8, 4), seed=seed))
        e_lr.append(rel(d, a @ b))
        e_dq4.append(rel(L.qgemm(a, b, 4, 4), a @ b))
    assert np.median(e_lr) > np.median(e_dq4)


def test_stage_timings_and_report_fields(L):
    """test_pipeline.py:203-221"""
    a = gen(20, 20, "uniform", 19)
    _, timings = L.lramm(a, a, L.LrammParams(rank=3, seed=20))
    assert sorted(timings.wall_ns) == sorted(["rsvd", "scaling", "gemm1", "gemm2", "gemm3"])
    assert all(v >= 0 for v in timings.wall_ns.values())
    assert isinstance(timings.macs, L.CostModel)
    a, b = gen(24, 24, "uniform", 21), gen(24, 24, "uniform", 22)
    d, report = L.evaluate(a, b, L.LrammParams(rank=4, bits=(8, 8, 4), seed=23))
    as_dict = report.to_dict()
    for key in ("m", "n", "k", "r", "d1", "d2", "d3", "q", "seed", "fro_error", "rel_error", "bound_combined",
                "macs", "wall_ns"):
        assert key in as_dict
    assert as_dict["macs"]["total"] == report.macs.total
    assert report.fro_error <= report.bound_combined
    assert d.shape == (24, 24)
    values, source = L.leading_sigmas(gen(30, 30, "uniform", 24), 5)
    assert source == "oracle" and len(values) == 5 and np.all(np.diff(values) <= 1e-12)


# ------------------------------------------------------------------ rsvd (test_rsvd.py)


def test_range_finder_contracts(L):
    """test_rsvd.py:34-63"""
    q = L.range_finder(np.eye(4), L.RsvdParams(rank=2, oversample=0, seed=1))
    assert q.shape == (4, 2) and np.linalg.norm(q.T @ q - np.eye(2)) <= 1e-8
    a = gen(60, 50, "lowrank", 2, 3)
    q = L.range_finder(a, L.RsvdParams(rank=3, oversample=2, seed=3))
    assert np.linalg.norm(a - q @ (q.T @ a)) <= 1e-8 * np.linalg.norm(a)
    a = gen(20, 15, "normal", 4)
    p = L.RsvdParams(rank=5, power_iters=1, oversample=3, seed=9)
    assert np.array_equal(L.range_finder(a, p), L.range_finder(a, p))
    with pytest.raises(L.ParameterError):
        L.range_finder(np.ones((4, 4)), L.RsvdParams(rank=5))
    assert L.range_finder(np.eye(6), L.RsvdParams(rank=4, oversample=50, seed=1)).shape == (6, 6)


def test_rsvd_rank_one_orthonormal_deterministic(L):
    """test_rsvd.py:68-111"""
    u = np.zeros((30, 1))
    u[4, 0] = 1.0
    v = np.zeros((20, 1))
    v[11, 0] = 1.0
    a = 3.0 * u @ v.T
    f = L.rsvd(a, L.RsvdParams(rank=1, seed=5))
    assert abs(float(f.sigma[0]) - 3.0) <= 1e-8 and np.linalg.norm(a - f.reconstruct()) <= 1e-8
    a = gen(40, 30, "uniform", 6)
    f = L.rsvd(a, L.RsvdParams(rank=8, seed=7))
    assert np.linalg.norm(f.u.T @ f.u - np.eye(8)) <= 1e-8 * math.sqrt(8)
    assert np.linalg.norm(f.v.T @ f.v - np.eye(8)) <= 1e-8 * math.sqrt(8)
    assert np.all(np.diff(f.sigma) <= 1e-12)
    a = gen(25, 25, "normal", 8)
    f1, f2 = L.rsvd(a, L.RsvdParams(rank=5, seed=11)), L.rsvd(a, L.RsvdParams(rank=5, seed=11))
    assert np.array_equal(f1.u, f2.u) and np.array_equal(f1.sigma, f2.sigma) and np.array_equal(f1.v, f2.v)


def test_rsvd_diag_spectrum_recovery(L):
    """test_rsvd.py:87-102"""
    a = np.diag([5.0, 4.0, 3.0, 2.0, 1.0])
    errs = [float(np.max(np.abs(L.rsvd(a, L.RsvdParams(rank=2, power_iters=1, oversample=2, seed=s)).sigma
                               - [5.0, 4.0]))) for s in range(10)]
    assert np.median(errs) <= 5e-2
    for s in range(5):
        f = L.rsvd(a, L.RsvdParams(rank=2, power_iters=4, oversample=2, seed=s))
        assert np.max(np.abs(f.sigma - [5.0, 4.0])) <= 1e-6
    f = L.rsvd(a, L.RsvdParams(rank=2, power_iters=1, seed=0))
    assert np.max(np.abs(f.sigma - [5.0, 4.0])) <= 1e-10


def test_rsvd_spectral_error_bound_and_power_iterations(L):
    """test_rsvd.py:114-138"""
    a_by_seed = [gen(100, 100, "uniform", 500 + s) for s in range(20)]
    errs = [np.linalg.norm(a - L.rsvd(a, L.RsvdParams(rank=10, seed=s)).reconstruct(), 2)
            for s, a in enumerate(a_by_seed)]
    sigma11 = max(float(L.oracle_svd(a).sigma[10]) for a in a_by_seed)
    assert np.mean(errs) <= L.rsvd_error_bound(sigma11, 100, 10, 0)
    r0, r2 = [], []
    for seed in range(20):
        a = gen(60, 60, "normal", 600 + seed)
        r0.append(np.linalg.norm(a - L.rsvd(a, L.RsvdParams(rank=6, power_iters=0, seed=seed)).reconstruct()))
        r2.append(np.linalg.norm(a - L.rsvd(a, L.RsvdParams(rank=6, power_iters=2, seed=seed)).reconstruct()))
    assert np.median(r2) <= np.median(r0)


def test_truncation_contracts(L):
    """test_rsvd.py:141-178"""
    a = np.diag([3.0, 2.0, 1.0])
    assert abs(np.linalg.norm(a - L.truncate_svd(L.oracle_svd(a), 2).reconstruct()) - 1.0) <= 1e-12
    a = gen(10, 10, "normal", 9)
    assert np.linalg.norm(a - L.truncate_svd(L.oracle_svd(a), 10).reconstruct()) <= 1e-10 * np.linalg.norm(a)
    a = gen(50, 40, "normal", 10)
    f = L.oracle_svd(a)
    err = np.linalg.norm(a - L.truncate_svd(f, 10).reconstruct())
    assert abs(err - math.sqrt(float(np.sum(f.sigma[10:] ** 2)))) <= 1e-8 * np.linalg.norm(a)
    for seed in range(6):
        a = gen(30, 24, "uniform", 40 + seed)
        f = L.oracle_svd(a)
        for rank in (2, 5, 12):
            err = np.linalg.norm(a - L.truncate_svd(f, rank).reconstruct())
            assert err <= L.svd_trunc_bound(float(f.sigma[rank]), 24, rank) + 1e-12
    with pytest.raises(L.ParameterError):
        L.truncate_svd(L.oracle_svd(np.eye(4)), 5)


def test_quantized_svd_contracts(L):
    """test_rsvd.py:183-241"""
    _, _, rec = L.quantized_svd_approx(np.diag([2.0, 1.0]), 2, 24, 24)
    assert np.linalg.norm(rec - np.diag([2.0, 1.0])) <= 1e-4 * math.sqrt(5.0)
    a = gen(40, 40, "uniform", 12)
    qu, qv, _ = L.quantized_svd_approx(a, 6, 8, 8)
    assert np.max(np.abs(qu.data)) <= 127 and np.max(np.abs(qv.data)) <= 127
    errs = [rel(L.quantized_svd_approx(a1, 1, 8, 8)[2], a1)
            for a1 in (gen(32, 32, "lowrank", 700 + s, 1) for s in range(20))]
    assert np.mean(errs) <= 0.02
    sq, bound = [], None
    for seed in range(20):
        a = gen(64, 64, "lowrank", 800 + seed, 8)
        f = L.oracle_svd(a)
        sq.append(np.linalg.norm(a - L.quantized_svd_approx(a, 8, 8, 8)[2]) ** 2)
        bound = L.qsvd_bound(L.BoundInputs(m=64, n=64, r=8, sigma1=float(f.sigma[0]), sigma_r1=float(f.sigma[8]),
                                           d1=8, d2=8))
    assert np.mean(sq) <= bound
    a = gen(20, 14, "normal", 13)
    qu, qv, rec = L.quantized_svd_approx(a, 5, 16, 16)
    assert np.allclose(rec, L.dequantize(qu) @ L.dequantize(qv).T, rtol=0, atol=1e-12)


# ------------------------------------------------------------------ quant (test_quant.py)


def test_qgemm_reference_contracts(L):
    """test_quant.py:157-224"""
    assert L.qgemm(np.array([[1.0]]), np.array([[1.0]]), 8, 8)[0, 0] == 1.0
    b = np.array([[1.0, -64 / 127], [5 / 127, 100 / 127]])
    assert np.max(np.abs(L.qgemm(np.eye(2), b, 8, 8) - b)) <= 1e-15
    a, b = gen(64, 64, "uniform", 81), gen(64, 64, "uniform", 82)
    err = np.linalg.norm(L.qgemm(a, b, 8, 8) - a @ b)
    qa, qb = L.quantize(a, 8), L.quantize(b, 8)
    bound = L.qgemm_bound(L.BoundInputs(m=64, n=64, k=64, sigma1=np.linalg.norm(a, 2), gamma1=np.linalg.norm(b, 2),
                                        lambda1=qa.scale, lambda2=qb.scale))
    assert err <= bound
    a = gen(96, 96, "normal", 86)
    a /= np.max(np.abs(a))
    b = gen(96, 96, "normal", 87)
    b /= np.max(np.abs(b))
    assert rel(L.qgemm(a, b, 24, 24), a @ b) <= 1e-5
    e4, e8 = [], []
    for seed in range(30):
        a, b = gen(128, 128, "uniform", 9000 + seed), gen(128, 128, "uniform", 9500 + seed)
        e4.append(rel(L.qgemm(a, b, 4, 4), a @ b))
        e8.append(rel(L.qgemm(a, b, 8, 8), a @ b))
    assert np.median(e8) < np.median(e4)
    a = gen(16, 16, "binary", 90)
    assert np.array_equal(L.dequantize(L.quantize(a, 8)), a)
