"""The tile Cholesky behind CholeskyQR (lramm_cholqr_pass) on the B200.

The reference factors its sketches with numpy/LAPACK (rsvd.py range_finder -> np.linalg.qr);
our CholeskyQR must produce the same Q and report a breakdown exactly where LAPACK's
potrf would (info = first failing column + 1), for every position of the failing column in
the two-column POTRF steps and 32-column tiles, and stay exact under extreme scaling (the
POTRF prescales each diagonal tile by a power of 4).
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def dev():
    return torch.device("cuda", 0)


def cholqr_pass(y):
    from paper_2405_16917_b200 import _native as N
    from paper_2405_16917_b200._device import WORKSPACE, ptr, stream_handle

    m, w = y.shape
    y = y.contiguous()
    gram = y.T @ y
    q = torch.empty((m, w), dtype=torch.float64, device=y.device)
    lo = torch.zeros((w, w), dtype=torch.float64, device=y.device)
    info = torch.zeros(1, dtype=torch.int32, device=y.device)
    wsz = N.LIB.lramm_cholqr_pass_ws(m, w)
    ws = WORKSPACE.get(wsz, y.device)
    N.check(N.LIB.lramm_cholqr_pass(ptr(y), m, w, w, ptr(gram.contiguous()), ptr(q), w, ptr(lo), ptr(info), ptr(ws),
                                    wsz, stream_handle(y.device)))
    torch.cuda.synchronize()
    return q.cpu().numpy(), lo.cpu().numpy(), int(info.item()), gram.cpu().numpy()


@pytest.mark.parametrize("w", [1, 2, 3, 31, 32, 33, 63, 64, 65, 100, 272, 527])
def test_cholesky_matches_lapack(w):
    rng = np.random.default_rng(w)
    y = rng.standard_normal((max(2 * w, 64), w)) @ np.diag(np.linspace(1.0, 4.0, w))
    q, lo, info, gram = cholqr_pass(torch.from_numpy(y).to(dev()))
    assert info == 0
    ref = np.linalg.cholesky(gram)
    assert np.max(np.abs(np.tril(lo) - ref)) <= 1e-12 * np.max(np.abs(ref))
    assert np.linalg.norm(q.T @ q - np.eye(w)) <= 1e-10 * np.sqrt(w)


@pytest.mark.parametrize("j", [1, 2, 3, 30, 31, 32, 33, 62, 63, 64, 65, 100])
def test_cholesky_breakdown_column(j):
    """Column j a copy of column 0: the Schur complement at j is rounding noise -> info = j + 1."""
    w = 128
    rng = np.random.default_rng(7 + j)
    y = rng.standard_normal((400, w))
    y[:, j] = y[:, 0]
    _, _, info, _ = cholqr_pass(torch.from_numpy(y).to(dev()))
    assert info == j + 1


@pytest.mark.parametrize("scale", [1e-150, 2.0**-500, 1e-30, 1e30, 2.0**480, 1e150])
def test_cholesky_extreme_scales(scale):
    w = 100
    rng = np.random.default_rng(3)
    y0 = rng.standard_normal((300, w))
    q0, lo0, info0, _ = cholqr_pass(torch.from_numpy(y0).to(dev()))
    q, lo, info, gram = cholqr_pass(torch.from_numpy(y0 * scale).to(dev()))
    assert info0 == 0 and info == 0
    ref = np.linalg.cholesky(gram)
    assert np.max(np.abs(np.tril(lo) - ref)) <= 1e-12 * np.max(np.abs(ref))
    assert np.max(np.abs(q - q0)) <= 1e-12


@pytest.mark.gpu
@pytest.mark.parametrize("m,n", [(600, 138), (1200, 272), (2000, 544), (3000, 1056)])
def test_svd_eig_preconditioned_deterministic_and_accurate(m, n):
    # the eigenvector-preconditioned SVD (tridiagonalisation pushes, bisection, twisted
    # factorisations, back-transform, gated Jacobi) is free of atomics and races: bitwise equal
    # over repeated calls.  It is normwise backward stable, like LAPACK gesdd (the reference's
    # NumPy backend, _pure.py:29-35): sigma errors ~ eps sigma_1 sqrt(n) (the graded inputs here
    # reach kappa = 6e4 at n = 1056, where one-sided Jacobi is relatively accurate instead)
    import torch

    from paper_2405_16917_b200 import _native as N
    from paper_2405_16917_b200._device import WORKSPACE, ptr, stream_handle

    g = np.random.default_rng(n)
    a_h = g.standard_normal((m, n)) * np.exp(-np.arange(n) / 96.0)
    a = torch.tensor(a_h, device="cuda")
    outs = []
    for _ in range(2):
        u = torch.empty(m, n, dtype=torch.float64, device="cuda")
        s = torch.empty(n, dtype=torch.float64, device="cuda")
        v = torch.empty(n, n, dtype=torch.float64, device="cuda")
        info = torch.zeros(4, dtype=torch.int32, device="cuda")
        wsz = N.LIB.lramm_svd_ws(m, n)
        ws = WORKSPACE.get(wsz, torch.device("cuda"))
        N.check(N.LIB.lramm_svd(ptr(a), m, n, ptr(u), ptr(s), ptr(v), ptr(info), ptr(ws), wsz, stream_handle()))
        torch.cuda.synchronize()
        outs.append((u.cpu().numpy(), s.cpu().numpy(), v.cpu().numpy()))
    for x, y in zip(outs[0], outs[1]):
        assert np.array_equal(x, y)
    u, s, v = outs[0]
    s_ref = np.linalg.svd(a_h, compute_uv=False)
    assert np.max(np.abs(s - s_ref)) <= 1e-13 * s_ref[0]
    assert np.max(np.abs(s - s_ref)[s_ref > 1e-3 * s_ref[0]] / s_ref[s_ref > 1e-3 * s_ref[0]]) <= 1e-12
    assert np.max(np.abs(v.T @ v - np.eye(n))) <= 1e-13
    assert np.linalg.norm((u * s) @ v.T - a_h) <= 1e-12 * np.linalg.norm(a_h)
