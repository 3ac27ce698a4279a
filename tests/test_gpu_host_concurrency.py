"""Concurrent host callers of the drop-in entry point (`lramm(numpy)` -> `lramm_host_lramm`).

The reference's kernels are thread-safe and its sweeps call them from a thread pool
(`cli.py:415-419`); the host C ABI leases one context per call, submits each call's uploads as a
unit, queues the factorisations of large products in arrival order on the device and brings D
and the status word down on a download stream.  Results must not depend on what else is in
flight: every concurrent call is bitwise equal to the same call made alone.
"""

from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def L():
    import paper_2405_16917_b200 as pkg

    return pkg


def _pairs(m, k, n, count, dtype):
    rng = np.random.default_rng(20240516)
    out = []
    for _ in range(count):
        u = rng.standard_normal((m, 24)) * (np.arange(1, 25) ** -1.0)
        a = (u @ rng.standard_normal((24, k))).astype(dtype)
        b = (rng.standard_normal((k, 24)) @ rng.standard_normal((24, n))).astype(dtype)
        out.append((a, b))
    return out


@pytest.mark.parametrize("shape,mode", [((96, 4096, 80), "fast"),      # max dim >= 4096: device-side FIFO of the calls
                                        ((192, 160, 176), "parity"),   # small: calls run side by side
                                        ((128, 4100, 64), "parity")])
def test_concurrent_host_calls_match_isolated_calls(L, shape, mode):
    m, k, n = shape
    pairs = _pairs(m, k, n, 3, np.float32 if mode == "fast" else np.float64)
    params = [L.LrammParams(rank=16, bits=(8, 8, 8), seed=s, mode=mode, power_iters=1,
                            **({"granularity": "row", "sketch_bits": 8, "power_bits": 8, "proj_bits": 8}
                               if mode == "fast" else {})) for s in (3, 4)]
    jobs = [(pa, pr) for pa in pairs for pr in params] * 3
    alone = {}
    for i, ((a, b), p) in enumerate(jobs[: len(pairs) * len(params)]):
        alone[i] = L.lramm(a, b, p)[0].copy()

    def call(i):
        (a, b), p = jobs[i]
        d, t = L.lramm(a, b, p)
        assert set(t.wall_ns) == {"rsvd", "scaling", "gemm1", "gemm2", "gemm3"}
        assert all(v >= 0 for v in t.wall_ns.values())
        return i, d

    with ThreadPoolExecutor(max_workers=6) as pool:
        for i, d in pool.map(call, range(len(jobs))):
            ref = alone[i % len(alone)]
            assert d.dtype == ref.dtype and np.array_equal(d, ref), f"call {i} differs from the isolated call"


def test_concurrent_failure_does_not_poison_other_calls(L):
    """A call that fails on the device (non-finite input, pipeline.py:177-181) raises in its own
    thread; the calls around it return their usual results and the contexts stay usable."""
    (a, b), (a2, b2) = _pairs(64, 4096, 72, 2, np.float64)
    bad = a.copy()
    bad[5, 7] = np.inf
    p = L.LrammParams(rank=8, bits=(8, 8, 8), seed=1)
    good = L.lramm(a2, b2, p)[0].copy()

    def call(i):
        if i % 3 == 1:
            with pytest.raises((L.ParameterError, RuntimeError)):
                L.lramm(bad, b, p)
            return None
        return L.lramm(a2, b2, p)[0]

    with ThreadPoolExecutor(max_workers=4) as pool:
        for d in pool.map(call, range(12)):
            if d is not None:
                assert np.array_equal(d, good)
    assert np.array_equal(L.lramm(a2, b2, p)[0], good)
