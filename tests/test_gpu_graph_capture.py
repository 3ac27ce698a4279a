"""`lramm_device` captured into a CUDA graph (how `bench.py` times it) against the eager call.

While a stream is being captured the rarely taken branches of the factorisations (second
CholeskyQR pass, refinement of the small SVD's preconditioner) are recorded as IF nodes of the
graph (CUDA conditional nodes, `CondIf` in csrc/common.cuh) instead of sequences of self-gating
kernels.  The replayed graph must give the eager result bit for bit both when the branches are
skipped (well-conditioned sketches, the benchmarked case) and when they are taken: a
rank-deficient operand breaks the first Cholesky, which forces the second pass (and then the
Householder fallback), and a clustered spectrum sends the small SVD through its Jacobi fallback.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def L():
    import paper_2405_16917_b200 as pkg

    return pkg


def _inputs(kind, m, k, n, dtype):
    rng = np.random.default_rng(11)
    if kind == "decaying":
        t = min(m, k, n)
        sig = np.exp(-np.arange(t) / 12.0) + 1e-4
        a = (np.linalg.qr(rng.standard_normal((m, t)))[0] * sig) @ np.linalg.qr(rng.standard_normal((k, t)))[0].T
        b = (np.linalg.qr(rng.standard_normal((k, t)))[0] * sig) @ np.linalg.qr(rng.standard_normal((n, t)))[0].T
    elif kind == "rank_deficient":  # rank 3 < sketch width: singular Gram matrices
        a = rng.standard_normal((m, 3)) @ rng.standard_normal((3, k))
        b = rng.standard_normal((k, 3)) @ rng.standard_normal((3, n))
    else:  # "clustered": many equal singular values
        a = np.linalg.qr(rng.standard_normal((m, k)))[0] if m >= k else np.linalg.qr(rng.standard_normal((k, m)))[0].T
        b = np.linalg.qr(rng.standard_normal((k, n)))[0] if k >= n else np.linalg.qr(rng.standard_normal((n, k)))[0].T
    return a.astype(dtype), b.astype(dtype)


@pytest.mark.parametrize("kind", ["decaying", "rank_deficient", "clustered"])
@pytest.mark.parametrize("mode,gran", [("fast", "row"), ("fast", "tensor"), ("parity", "tensor")])
def test_graph_replay_equals_eager(L, kind, mode, gran):
    m, k, n = 320, 288, 304
    dev = torch.device("cuda", 0)
    a, b = _inputs(kind, m, k, n, np.float32 if mode == "fast" else np.float64)
    ta, tb = torch.from_numpy(a).to(dev), torch.from_numpy(b).to(dev)
    kw = dict(rank=24, bits=(8, 8, 8), power_iters=1, oversample=8, seed=2, mode=mode, granularity=gran)
    if mode == "fast":
        kw.update(sketch_bits=8, power_bits=8, proj_bits=8)
    p = L.LrammParams(**kw)
    eager, st, _ = L.lramm_device(ta, tb, p)
    torch.cuda.synchronize()
    assert int(st.item()) == 0
    eager = eager.clone()
    out = torch.empty_like(eager)
    s = torch.cuda.Stream(device=dev)
    s.wait_stream(torch.cuda.current_stream(dev))
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        L.lramm_device(ta, tb, p, out=out)  # sizes this stream's workspace before the capture
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=s):
            _o, status, _t = L.lramm_device(ta, tb, p, out=out)
    torch.cuda.synchronize()
    for _ in range(2):
        out.zero_()
        g.replay()
        torch.cuda.synchronize()
        assert int(status.item()) == 0
        assert torch.equal(out, eager), f"graph replay differs from the eager call ({kind}, {mode}, {gran})"
    assert torch.isfinite(out).all()
