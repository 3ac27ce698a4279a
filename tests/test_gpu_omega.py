"""Device Omega generator vs NumPy (matcore.py:89-92, rsvd.py:56): bitwise."""
import time

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _key(seed, n, w):
    ss = np.random.SeedSequence([int(seed) & 0xFFFFFFFFFFFFFFFF, 0x534B, n, w])
    k = np.random.Philox(ss).state["state"]["key"]
    return int(k[0]), int(k[1])


def _device(seed, n, w):
    from paper_2405_16917_b200 import _native as N
    from paper_2405_16917_b200._device import WORKSPACE, ptr, stream_handle

    dev = torch.device("cuda", 0)
    out = torch.empty((n, w), dtype=torch.float64, device=dev)
    wsz = N.LIB.lramm_omega_ws(n, w)
    ws = WORKSPACE.get(wsz, dev)
    k0, k1 = _key(seed, n, w)
    N.check(N.LIB.lramm_omega(k0, k1, n, w, ptr(out), ptr(ws), wsz, stream_handle(dev)))
    return out.cpu().numpy()


@pytest.mark.parametrize("seed,n,w", [(0, 1, 1), (3, 7, 5), (12345, 1024, 74), (2**63 + 5, 4096, 272),
                                      (99, 333, 1)])
def test_omega_bitwise_vs_numpy(seed, n, w):
    ref = np.random.Generator(np.random.Philox(np.random.SeedSequence(
        [int(seed) & 0xFFFFFFFFFFFFFFFF, 0x534B, n, w]))).standard_normal((n, w))
    got = _device(seed, n, w)
    assert np.array_equal(got, ref)


def test_omega_large_with_many_tail_draws():
    """c5 width: 8.6 M draws, ~2,000 through the ziggurat tail."""
    n, w, seed = 8192, 1056, 7
    ref = np.random.Generator(np.random.Philox(np.random.SeedSequence([seed, 0x534B, n, w]))).standard_normal((n, w))
    t0 = time.perf_counter()
    got = _device(seed, n, w)
    assert np.array_equal(got, ref)
    assert np.sum(np.abs(ref) > 3.6541528853610088) > 100  # tail values were exercised
