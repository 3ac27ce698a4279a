"""Kernel-level parity on the B200 against the CPU oracle (bit-exact for integer work).

Mirrors the reference's kernel tests (pkg/tests/test_backends.py, test_quant.py):
quantiser KATs and bit-identity, exact integer products, qgemm dequantisation,
fp64 GEMM, thin QR and the Jacobi SVD contracts.
"""

import ctypes

import numpy as np
import pytest

import lramm_oracle as O

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def L():
    import paper_2405_16917_b200 as lib

    return lib


@pytest.fixture(scope="module")
def N():
    from paper_2405_16917_b200 import _native

    return _native


def dev():
    return torch.device("cuda", 0)


# ------------------------------------------------------------------ quantiser


def test_quantize_kats(L):
    q = L.quantize(np.array([[1.0, -1.0]]), 8)  # test_quant.py:32-35
    assert q.scale == 127.0 and q.data.tolist() == [[127, -127]]
    q = L.quantize(np.array([[2.0, 0.0]]), 4)  # :38-41
    assert q.scale == 3.5 and q.data.tolist() == [[7, 0]]
    q = L.quantize(np.zeros((2, 2)), 8)  # :44-47
    assert q.scale == 1.0 and not q.data.any()
    with pytest.raises(L.ParameterError):
        L.quantize(np.array([[1.0, np.nan]]), 8)  # :60-62
    with pytest.raises(L.ParameterError):
        L.quantize(np.ones((2, 2)), 25)


def test_scale_round_clip_half_to_even(L):
    from paper_2405_16917_b200 import kernels

    halves = np.array([[0.5, 1.5, 2.5, -0.5, -1.5, -2.5]])  # test_backends.py:46-51
    assert kernels.scale_round_clip(halves, 1.0, 127).tolist() == [[0, 2, 2, 0, -2, -2]]
    a = O.generate(29, 17, "uniform", 4) * 2.0 - 1.0
    assert np.array_equal(kernels.scale_round_clip(a, 127.0, 127), O.scale_round_clip(a, 127.0, 127))


@pytest.mark.parametrize("bits", [2, 3, 4, 5, 8, 12, 16, 24])
@pytest.mark.parametrize("shape", [(33, 47), (1, 300), (257, 5)])
def test_quantize_bit_exact(L, bits, shape):
    x = O.generate(*shape, "normal", 100 + bits)
    q = L.quantize(x, bits)
    d, s = O.quantize_tensor(x, bits)
    assert q.scale == s
    assert np.array_equal(q.data, d)


def test_quantize_fp32_input_bit_exact(L):
    x = O.synth(64, 96, "exp:8", 9, 0, 0)  # float32
    q = L.quantize(x, 8)
    d, s = O.quantize_tensor(x, 8)
    assert q.scale == s and np.array_equal(q.data, d)


@pytest.mark.parametrize("gran", ["row", "col"])
@pytest.mark.parametrize("transpose", [False, True])
@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_quantize_granularity_layouts(N, gran, transpose, dtype):
    from paper_2405_16917_b200.quant import quantize_device

    x = O.generate(77, 45, "normal", 5).astype(dtype)
    x[3] = 0.0
    x[:, 7] = 0.0
    t = torch.from_numpy(x).to(dev())
    code = N.GRAN_ROW if gran == "row" else N.GRAN_COL
    q, s, flag = quantize_device(t, 6, code, transpose, N.I8)
    d, sref = (O.quantize_rows if gran == "row" else O.quantize_cols)(x, 6)
    got = q.cpu().numpy().astype(np.int32)
    if transpose:
        got = got[:, :77].T
    else:
        got = got[:, :45]
    assert np.array_equal(got, d)
    assert np.array_equal(s.cpu().numpy(), sref)
    assert int(flag.item()) == 0
    # padding columns are zero
    pad = q.cpu().numpy()[:, (77 if transpose else 45):]
    assert not pad.any()


def _oracle_quant(x, bits, gran):
    if gran == "tensor":
        d, s = O.quantize_tensor(x, bits)
        return d, np.array([s])
    return (O.quantize_rows if gran == "row" else O.quantize_cols)(x, bits)


@pytest.mark.parametrize("shape", [(77, 45), (130, 300), (1, 5), (300, 1), (64, 64)])
@pytest.mark.parametrize("grans,bits", [(("tensor", "tensor"), (8, 8)), (("row", "col"), (8, 8)),
                                        (("row", "col"), (4, 8)), (("col", "tensor"), (6, 3)),
                                        (("row", "row"), (8, 8))])
@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("strided", [False, True])
def test_quantize_pair_bit_exact(N, shape, grans, bits, dtype, strided):
    """lramm_quantize_pair: both layouts equal two independent quantisations (quant.py:55-71)."""
    rows, cols = shape
    base = O.generate(rows, cols + (3 if strided else 0), "normal", rows + cols).astype(dtype)
    base[0, : min(cols, 4)] = 0.0
    x = base[:, :cols]
    t = torch.from_numpy(base).to(dev())[:, :cols]  # ld = cols + 3: the unvectorised path
    code = {"tensor": N.GRAN_TENSOR, "row": N.GRAN_ROW, "col": N.GRAN_COL}
    ldr, ldt = ((cols + 15) // 16) * 16, ((rows + 15) // 16) * 16
    qr = torch.full((rows, ldr), 99, dtype=torch.int8, device=dev())
    qt = torch.full((cols, ldt), 99, dtype=torch.int8, device=dev())
    ns = {"tensor": 1, "row": rows, "col": cols}
    sr = torch.empty(ns[grans[0]], dtype=torch.float64, device=dev())
    st = torch.empty(ns[grans[1]], dtype=torch.float64, device=dev())
    flag = torch.zeros(1, dtype=torch.int32, device=dev())
    wsz = N.LIB.lramm_quantize_ws(rows, cols)
    ws = torch.empty(wsz, dtype=torch.uint8, device=dev())
    vp = ctypes.c_void_p
    N.check(N.LIB.lramm_quantize_pair(vp(t.data_ptr()), N.F32 if dtype == np.float32 else N.F64, rows, cols,
                                      t.stride(0), bits[0], code[grans[0]], vp(qr.data_ptr()), ldr,
                                      vp(sr.data_ptr()), bits[1], code[grans[1]], vp(qt.data_ptr()), ldt,
                                      vp(st.data_ptr()), vp(flag.data_ptr()), vp(ws.data_ptr()), wsz,
                                      vp(torch.cuda.current_stream().cuda_stream)))
    dr, srf = _oracle_quant(x, bits[0], grans[0])
    dt, stf = _oracle_quant(x, bits[1], grans[1])
    got_r, got_t = qr.cpu().numpy(), qt.cpu().numpy()
    assert np.array_equal(got_r[:, :cols].astype(np.int32), dr)
    assert np.array_equal(got_t[:, :rows].T.astype(np.int32), dt)
    assert np.array_equal(sr.cpu().numpy(), srf) and np.array_equal(st.cpu().numpy(), stf)
    assert not got_r[:, cols:].any() and not got_t[:, rows:].any()
    assert int(flag.item()) == 0


def test_quantize_pair_nonfinite_flag(N):
    x = torch.ones((40, 70), dtype=torch.float32, device=dev())
    x[5, 9] = float("nan")
    qr = torch.empty((40, 80), dtype=torch.int8, device=dev())
    qt = torch.empty((70, 48), dtype=torch.int8, device=dev())
    s = torch.empty(2, dtype=torch.float64, device=dev())
    flag = torch.zeros(1, dtype=torch.int32, device=dev())
    wsz = N.LIB.lramm_quantize_ws(40, 70)
    ws = torch.empty(wsz, dtype=torch.uint8, device=dev())
    vp = ctypes.c_void_p
    N.check(N.LIB.lramm_quantize_pair(vp(x.data_ptr()), N.F32, 40, 70, 70, 8, N.GRAN_TENSOR, vp(qr.data_ptr()), 80,
                                      vp(s.data_ptr()), 8, N.GRAN_TENSOR, vp(qt.data_ptr()), 48,
                                      vp(s.data_ptr() + 8), vp(flag.data_ptr()), vp(ws.data_ptr()), wsz,
                                      vp(torch.cuda.current_stream().cuda_stream)))
    assert int(flag.item()) == 1


# ------------------------------------------------------------------ integer GEMM


@pytest.mark.parametrize("mnk", [(19, 11, 31), (128, 128, 128), (300, 272, 4096), (1, 16, 8), (513, 129, 1000)])
def test_imatmul_exact(mnk):
    from paper_2405_16917_b200 import kernels

    m, n, k = mnk
    rng = np.random.Generator(np.random.Philox(key=3))
    a = rng.integers(-127, 128, size=(m, k)).astype(np.int32)
    b = rng.integers(-127, 128, size=(k, n)).astype(np.int32)
    out = kernels.imatmul(a, b)
    assert out.dtype == np.int64
    assert np.array_equal(out, a.astype(np.int64) @ b.astype(np.int64))


@pytest.mark.parametrize("amp,k", [(255, 64), (40000, 500), (1 << 20, 1000), ((1 << 31) - 1, 2)])
def test_imatmul_multi_limb_exact(amp, k):
    """Entries beyond +-127: limb decomposition, exact int64 like _core.imatmul."""
    from paper_2405_16917_b200 import kernels

    rng = np.random.Generator(np.random.Philox(key=amp % 1000))
    a = rng.integers(-amp, amp, size=(33, k), endpoint=True).astype(np.int32)
    b = rng.integers(-amp, amp, size=(k, 45), endpoint=True).astype(np.int32)
    out = kernels.imatmul(a, b)
    assert np.array_equal(out, a.astype(np.int64) @ b.astype(np.int64))


def test_imatmul_extremes_and_shape_error():
    from paper_2405_16917_b200 import kernels

    a = np.full((130, 2048), -127, dtype=np.int32)
    b = np.full((2048, 40), 127, dtype=np.int32)
    assert np.all(kernels.imatmul(a, b) == -127 * 127 * 2048)
    with pytest.raises(ValueError, match="inner dimensions differ"):
        kernels.imatmul(a, a)


@pytest.mark.parametrize("split", [2, 5])
def test_igemm_split_k_exact(N, split):
    from paper_2405_16917_b200.quant import quantize_device

    m, n, k = 200, 96, 3000
    rng = np.random.default_rng(7)
    a = rng.integers(-127, 128, size=(m, k)).astype(np.int8)
    bt = rng.integers(-127, 128, size=(n, k)).astype(np.int8)
    lda = ((k + 15) // 16) * 16
    ta = torch.zeros((m, lda), dtype=torch.int8, device=dev())
    tb = torch.zeros((n, lda), dtype=torch.int8, device=dev())
    ta[:, :k] = torch.from_numpy(a).to(dev())
    tb[:, :k] = torch.from_numpy(bt).to(dev())
    out = torch.zeros((m, n), dtype=torch.int32, device=dev())
    e = N.Epilogue()
    e.out_dtype, e.accumulate, e.out, e.ldo = N.I32, 1, out.data_ptr(), n
    rc = N.LIB.lramm_igemm(m, n, k, ctypes.c_void_p(ta.data_ptr()), lda, ctypes.c_void_p(tb.data_ptr()), lda,
                           ctypes.byref(e), split, ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
    N.check(rc)
    ref = a.astype(np.int64) @ bt.astype(np.int64).T
    assert np.array_equal(out.cpu().numpy(), ref)


@pytest.mark.parametrize("bits", [(8, 8), (4, 8), (6, 6), (2, 3)])
def test_qgemm_bitwise(L, bits):
    a = O.generate(21, 35, "uniform", 80 + bits[0])
    b = O.generate(35, 17, "normal", 90 + bits[1])
    assert np.array_equal(L.qgemm(a, b, *bits), O.qgemm(a, b, *bits))


def test_qgemm_alpha_beta_bitwise(L):
    a = O.generate(6, 5, "uniform", 83)
    b = O.generate(5, 7, "uniform", 84)
    c = O.generate(6, 7, "normal", 85)
    assert np.array_equal(L.qgemm(a, b, 8, 8, alpha=2.0, beta=3.0, c=c), O.qgemm(a, b, 8, 8, 2.0, 3.0, c))
    assert np.array_equal(L.qgemm(a, b, 8, 8, alpha=-0.5), O.qgemm(a, b, 8, 8, -0.5))


def test_qgemm_large_bitwise(L):
    a = O.generate(700, 1100, "normal", 1)
    b = O.generate(1100, 333, "normal", 2)
    assert np.array_equal(L.qgemm(a, b, 8, 8), O.qgemm(a, b, 8, 8))


def test_qgemm_errors(L):
    with pytest.raises(L.ShapeError):
        L.qgemm(np.ones((2, 3)), np.ones((2, 3)), 8, 8)
    with pytest.raises(L.OverflowRiskError):
        L.qgemm(np.ones((1, (1 << 17) + 1)), np.ones(((1 << 17) + 1, 1)), 24, 24)


@pytest.mark.parametrize("bits", [(12, 12), (16, 16), (24, 24), (16, 8), (24, 12), (9, 3)])
def test_qgemm_bitwise_limbs(L, bits):
    """Bit budgets 9..24 (quant.py:16-28): 8-bit limb products, exact int64 accumulation."""
    a = O.generate(37, 300, "normal", 60 + bits[0])
    b = O.generate(300, 29, "uniform", 70 + bits[1])
    assert np.array_equal(L.qgemm(a, b, *bits), O.qgemm(a, b, *bits))
    c = O.generate(37, 29, "normal", 5)
    assert np.array_equal(L.qgemm(a, b, *bits, alpha=1.5, beta=-2.0, c=c), O.qgemm(a, b, *bits, 1.5, -2.0, c))


def test_qgemm_long_k_exact(L):
    """K * 127^2 >= 2^31: the single int8 product would overflow int32; the limb path chunks K."""
    k = 140000
    a = O.generate(3, k, "normal", 1)
    b = O.generate(k, 2, "normal", 2)
    assert np.array_equal(L.qgemm(a, b, 8, 8), O.qgemm(a, b, 8, 8))


def test_integer_matmul_and_dequantize(L):
    a = O.generate(8, 8, "normal", 71)
    b = O.generate(8, 8, "normal", 72)
    qa, qb = L.quantize(a, 8), L.quantize(b, 8)
    out = L.integer_matmul(qa, qb)
    assert out.dtype == np.int64
    assert np.array_equal(out, O.imatmul(*[O.quantize_tensor(x, 8)[0] for x in (a, b)]))
    d = L.dequantize(qa)
    assert np.array_equal(d, O.dequantize(*O.quantize_tensor(a, 8)))


@pytest.mark.parametrize("bits,k", [(8, 300), (16, 1000), (24, 70000)])
def test_integer_matmul_device_tensors(L, bits, k):
    # CUDA-tensor operands stay on the device (limb planes + exact int64 epilogue), bit-exact
    import torch

    a = O.generate(9, k, "normal", 81)
    b = O.generate(k, 7, "normal", 82)
    qa, qb = L.quantize(torch.tensor(a, device="cuda"), bits), L.quantize(torch.tensor(b, device="cuda"), bits)
    out = L.integer_matmul(qa, qb)
    assert out.is_cuda and out.dtype == torch.int64
    ref = O.imatmul(*[O.quantize_tensor(x, bits)[0] for x in (a, b)])
    assert np.array_equal(out.cpu().numpy(), ref)


# ------------------------------------------------------------------ fp64 building blocks


@pytest.mark.parametrize("mkn", [(37, 23, 41), (300, 700, 129), (4096, 64, 80)])
def test_dgemm_matches_blas(mkn):
    from paper_2405_16917_b200 import kernels

    m, k, n = mkn
    a = O.generate(m, k, "normal", 1)
    b = O.generate(k, n, "normal", 2)
    got = kernels.matmul(a, b)
    ref = a @ b
    assert np.max(np.abs(got - ref)) <= 1e-12 * (np.max(np.abs(ref)) + 1.0) * np.sqrt(k)


def test_dgemm_transposed_split_k(N):
    from paper_2405_16917_b200.rsvd import _dgemm

    a = O.generate(5000, 70, "normal", 3)
    b = O.generate(5000, 90, "normal", 4)
    got = _dgemm(1, torch.from_numpy(a).to(dev()), torch.from_numpy(b).to(dev()), 70, 90, 5000).cpu().numpy()
    ref = a.T @ b
    assert np.max(np.abs(got - ref)) <= 1e-12 * np.max(np.abs(ref)) * 10
    got2 = _dgemm(1, torch.from_numpy(a).to(dev()), torch.from_numpy(b).to(dev()), 70, 90, 5000).cpu().numpy()
    assert np.array_equal(got, got2)  # deterministic split-K


@pytest.mark.parametrize("mw", [(200, 16), (4096, 272), (1000, 74), (333, 100), (2048, 544), (3000, 1056)])
def test_qr_orthonormal_and_spans(mw):
    from paper_2405_16917_b200.rsvd import _qr_device

    m, w = mw
    y = O.synth(m, w, "exp:40", 5, 0, 0).astype(np.float64) @ np.diag(np.linspace(1, 3, w))
    q = _qr_device(torch.from_numpy(y).to(dev())).cpu().numpy()
    assert np.linalg.norm(q.T @ q - np.eye(w)) <= 1e-12 * np.sqrt(w)
    qh = np.linalg.qr(y)[0]
    # same column-nested basis as Householder up to column signs
    sign = np.sign(np.sum(q * qh, axis=0))
    assert np.max(np.abs(q * sign - qh)) <= 1e-10


@pytest.mark.parametrize("mw", [(2400, 544), (2200, 520), (2304, 576), (4400, 1056), (9000, 272), (4500, 1040)])
def test_qr_explicit_inverse_path(mw):
    """Tall sketches (w >= 512 with m >= 4 w, or w >= 256 with m >= 32 w) take Q = Y L^-T as the
    tile-doubling triangular inverse + one DMMA GEMM (factor.cu trinv_tiles_kernel): full and
    partial last tiles, odd tile counts, and the widest sketch (33 tiles)."""
    from paper_2405_16917_b200.rsvd import _qr_device

    m, w = mw
    y = O.synth(m, w, "exp:40", 7, 0, 0).astype(np.float64) @ np.diag(np.linspace(1, 3, w))
    q = _qr_device(torch.from_numpy(y).to(dev())).cpu().numpy()
    assert np.all(np.isfinite(q))
    assert np.linalg.norm(q.T @ q - np.eye(w)) <= 1e-12 * np.sqrt(w)
    qh = np.linalg.qr(y)[0]
    sign = np.sign(np.sum(q * qh, axis=0))
    assert np.max(np.abs(q * sign - qh)) <= 1e-10
    q2 = _qr_device(torch.from_numpy(y).to(dev())).cpu().numpy()
    assert np.array_equal(q, q2)  # deterministic


def test_qr_rank_deficient_falls_back_to_householder():
    from paper_2405_16917_b200.rsvd import _qr_device

    u = np.zeros((30, 1))
    u[4, 0] = 1.0
    y = u @ np.ones((1, 11))  # rank 1, width 11 (test_rsvd.py:68-76 shape)
    q = _qr_device(torch.from_numpy(y).to(dev())).cpu().numpy()
    assert np.linalg.norm(q.T @ q - np.eye(11)) <= 1e-10
    assert np.linalg.norm(y - q @ (q.T @ y)) <= 1e-12


@pytest.mark.parametrize("shape", [(20, 20), (35, 14), (14, 35), (300, 74), (4096, 272), (1000, 138), (90, 520),
                                   (1200, 544), (1100, 1056)])
def test_svd_contracts(shape):
    from paper_2405_16917_b200 import kernels

    a = O.generate(*shape, "normal", 5)
    u, s, v = kernels.svd(a)
    t = min(shape)
    sref = np.linalg.svd(a, compute_uv=False)
    assert u.shape == (shape[0], t) and v.shape == (shape[1], t)
    assert np.all(np.diff(s) <= 1e-12 * s[0])
    assert np.max(np.abs(s - sref)) <= 1e-10 * sref[0]
    assert np.linalg.norm(u.T @ u - np.eye(t)) <= 1e-8 * np.sqrt(t)
    assert np.linalg.norm(v.T @ v - np.eye(t)) <= 1e-8 * np.sqrt(t)
    assert np.linalg.norm(a - (u * s) @ v.T) <= 1e-10 * np.linalg.norm(a)


def test_svd_matches_reference_jacobi_golden():
    import os

    from paper_2405_16917_b200 import kernels

    G = np.load(os.path.join(os.path.dirname(__file__), "golden", "reference_golden.npz"))
    for shape in ((20, 20), (35, 14), (14, 35)):
        a = O.generate(*shape, "normal", 5)
        u, s, v = kernels.svd(a)
        key = f"jac_{shape[0]}x{shape[1]}"
        assert np.max(np.abs(s - G[key + "_s"])) <= 1e-12 * s[0]
        sign = np.sign(np.sum(u * G[key + "_u"], axis=0))
        assert np.max(np.abs(u * sign - G[key + "_u"])) <= 1e-9
        assert np.max(np.abs(v * sign - G[key + "_v"])) <= 1e-9


def test_svd_rank_deficient_completion():
    from paper_2405_16917_b200 import kernels

    a = O.generate(40, 12, "lowrank", 3, rank=3)
    u, s, v = kernels.svd(a)
    assert np.linalg.norm(u.T @ u - np.eye(12)) <= 1e-8
    assert np.linalg.norm(v.T @ v - np.eye(12)) <= 1e-8
    assert np.linalg.norm(a - (u * s) @ v.T) <= 1e-10 * np.linalg.norm(a)
