"""Ragged, tiny and degenerate shapes through the whole pipeline (both modes) vs the oracle."""
import numpy as np
import pytest

import lramm_oracle as O

pytestmark = pytest.mark.gpu

SHAPES = [
    ((2, 2, 2), 2),        # everything at the minimum rank
    ((3, 200, 2), 2),      # k >> m, n
    ((200, 3, 150), 2),    # sketch width clipped to k = 3
    ((37, 41, 43), 5),     # odd sizes, nothing a multiple of 16
    ((1000, 17, 900), 16),  # rank = min(k) - 1, very skinny inner dimension
    ((129, 513, 65), 33),  # tile-boundary straddlers
    ((64, 64, 64), 64),    # rank = min dim: w = r, no oversampling left
]


def _inputs(m, k, n, seed):
    a = O.generate(m, k, "normal", seed)
    b = O.generate(k, n, "uniform", seed + 1)
    return a, b


@pytest.mark.parametrize("shape,rank", SHAPES)
def test_parity_mode_edge_shapes(shape, rank):
    import paper_2405_16917_b200 as L

    m, k, n = shape
    a, b = _inputs(m, k, n, 3 * m + k)
    kw = dict(rank=rank, bits=(8, 8, 8), power_iters=1, seed=1)
    d, _ = L.lramm(a, b, L.LrammParams(**kw))
    assert d.shape == (m, n) and d.dtype == np.float64 and np.isfinite(d).all()
    ref = O.lramm(a, b, O.OracleParams(**kw))
    ref2 = O.lramm(a, b, O.OracleParams(**kw), svd_fn=O.jacobi_svd)
    tol = max(1e-3, 1.5 * O.rel_fro(ref2, ref))
    assert min(O.rel_fro(d, ref), O.rel_fro(d, ref2)) <= tol


@pytest.mark.parametrize("shape,rank", SHAPES)
@pytest.mark.parametrize("gran", ["tensor", "row"])
def test_fast_mode_edge_shapes(shape, rank, gran):
    import paper_2405_16917_b200 as L

    m, k, n = shape
    a, b = _inputs(m, k, n, 5 * m + n)
    a32, b32 = a.astype(np.float32), b.astype(np.float32)
    kw = dict(rank=rank, bits=(8, 8, 8), power_iters=1, seed=2)
    d, _ = L.lramm(a32, b32, L.LrammParams(**kw, mode="fast", sketch_bits=8, power_bits=8, proj_bits=8,
                                           granularity=gran))
    ref = O.lramm(a32, b32, O.OracleParams(**kw, spec=O.SketchSpec(8, 8, 8, gran)))
    ref2 = O.lramm(a32, b32, O.OracleParams(**kw, spec=O.SketchSpec(8, 8, 8, gran)), svd_fn=O.jacobi_svd)
    tol = max(1e-3, 1.5 * O.rel_fro(ref2, ref))
    assert min(O.rel_fro(d, ref), O.rel_fro(d, ref2)) <= tol


def test_device_and_host_paths_agree_on_ragged_shape():
    import torch

    import paper_2405_16917_b200 as L

    a, b = _inputs(131, 77, 95, 7)
    p = L.LrammParams(rank=9, bits=(8, 8, 4), power_iters=2, seed=4)
    d_host, _ = L.lramm(a, b, p)
    d_dev, _ = L.lramm(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda(), p)
    assert np.array_equal(d_dev.cpu().numpy(), d_host)


def test_concurrent_host_threads_are_safe():
    """The host entry points serialise on one device context (the plugin contract: thread-safe)."""
    import concurrent.futures as cf

    import paper_2405_16917_b200 as L

    a, b = _inputs(150, 120, 140, 9)
    p = L.LrammParams(rank=8, seed=3)
    ref, _ = L.lramm(a, b, p)
    with cf.ThreadPoolExecutor(max_workers=6) as ex:
        outs = list(ex.map(lambda _: L.lramm(a, b, p)[0], range(12)))
    assert all(np.array_equal(o, ref) for o in outs)
