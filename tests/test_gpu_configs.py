"""Parity at the BASELINE configurations' full shapes (BASELINE.json configs[0..3]).

The small-shape tests elsewhere pin semantics; these run the benchmarked code paths at the
sizes the bench measures, against the CPU oracle:

  * c2 (4096^3, r 256, p 16, q 1): parity mode vs the reference algorithm restated in NumPy
    (fp64 products, LAPACK QR / SVD, per-tensor QM recombination) at <= 1e-9 relative
    Frobenius (L4; the reference's own two backends agree to ~1e-13 here); fast mode
    (int8 per-row sketch / power / projection) vs the fast-mode restatement at <= 1e-3 (L5)
    and accuracy vs the exact product within 2 % of the reference algorithm's;
  * c3 (8192^3, r 512, p 32, q 2, poly 1.5): int4 packed sketch + int8 power / projection,
    per-row, vs the restatement at <= 1e-3 and accuracy within 2 %;
  * c1 fast mode and one c4 pair (2048^3, r 128, p 10, q 0, per-tensor int8) likewise;
  * the int8 tcgen05 GEMM's int32 accumulators bit-exact at the shapes whose code paths the
    small tests never reach: the two-CTA-per-SM shallow ring (c2 E3, 512 CTAs), the
    N-fastest rasterisation of an A beyond L2 (c3 int4 sketch, c5 int8 sketch 131072 x 1056
    x 8192), checked against exact products of sampled row blocks.

Inputs: the bench's seeded synthetic spectra, generated on the device.
"""

import ctypes

import numpy as np
import pytest

import lramm_oracle as O

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

CONFIGS = {
    "c1": dict(m=1024, k=1024, n=1024, rank=64, oversample=10, power_iters=1, spectrum=("exp", 32.0)),
    "c2": dict(m=4096, k=4096, n=4096, rank=256, oversample=16, power_iters=1, spectrum=("exp", 128.0)),
    "c3": dict(m=8192, k=8192, n=8192, rank=512, oversample=32, power_iters=2, spectrum=("poly", 1.5)),
    "c4": dict(m=2048, k=2048, n=2048, rank=128, oversample=10, power_iters=0, spectrum=("exp", 64.0)),
}
SPECS = {  # (sketch, power, proj bits, granularity) of the bench line for each config
    "c1": (8, 8, 8, "row"),
    "c2": (8, 8, 8, "row"),
    "c3": (4, 8, 8, "row"),
    "c4": (8, 8, 8, "tensor"),
}


@pytest.fixture(scope="module")
def L():
    import paper_2405_16917_b200 as lib

    return lib


def synth_pair(cfg, seed=0):
    """A = U diag(sigma) V^T, B likewise (Haar factors), stored fp32, generated on the device."""
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev)
    g.manual_seed(0x1A3A * 1000 + seed)
    kind, val = cfg["spectrum"]

    def mat(rows, cols):
        t = min(rows, cols)
        i = torch.arange(1, t + 1, device=dev, dtype=torch.float64)
        sig = i ** (-val) if kind == "poly" else torch.exp(-i / val) + 1e-4
        u, r = torch.linalg.qr(torch.randn(rows, t, generator=g, device=dev, dtype=torch.float64))
        u = u * torch.sign(torch.diagonal(r))
        v, r = torch.linalg.qr(torch.randn(cols, t, generator=g, device=dev, dtype=torch.float64))
        v = v * torch.sign(torch.diagonal(r))
        return ((u * sig) @ v.T).to(torch.float32).contiguous()

    return mat(cfg["m"], cfg["k"]), mat(cfg["k"], cfg["n"])


def rel_dev(x, ref):
    x, ref = x.double(), ref.double()
    return float(torch.linalg.norm(x - ref) / torch.linalg.norm(ref))


def run_fast(L, name, ta, tb):
    cfg = CONFIGS[name]
    sb, pb, jb, gran = SPECS[name]
    kw = dict(rank=cfg["rank"], bits=(8, 8, 8), power_iters=cfg["power_iters"], oversample=cfg["oversample"], seed=0)
    d, status, _ = L.lramm_device(ta, tb, L.LrammParams(**kw, mode="fast", sketch_bits=sb, power_bits=pb,
                                                        proj_bits=jb, granularity=gran))
    torch.cuda.synchronize()
    assert int(status.item()) == 0
    a, b = ta.cpu().numpy(), tb.cpu().numpy()
    ref = O.lramm(a, b, O.OracleParams(**kw, spec=O.SketchSpec(sb, pb, jb, gran)))
    par = O.lramm(a, b, O.OracleParams(**kw))  # the reference algorithm (parity mode)
    return d, torch.from_numpy(ref).to(d.device), torch.from_numpy(par).to(d.device)


@pytest.mark.parametrize("name", ["c1", "c2", "c4", "c3"])
def test_fast_mode_at_config_vs_restatement(L, name):
    """L5 at the bench shapes: the benchmarked fast-mode product vs the CPU restatement built from
    the reference's own quantiser semantics (<= 1e-3, the BASELINE bar), and its error vs the
    exact product within 2 % of the reference algorithm's error on the same inputs."""
    ta, tb = synth_pair(CONFIGS[name])
    d, ref, par = run_fast(L, name, ta, tb)
    assert rel_dev(d, ref) <= 1e-3, f"{name}: fast mode vs restatement {rel_dev(d, ref):.3e}"
    exact = ta.double() @ tb.double()
    e_ours, e_par = rel_dev(d, exact), rel_dev(par, exact)
    assert abs(e_ours - e_par) <= 0.02 * e_par, f"{name}: error vs exact {e_ours:.5f} vs reference {e_par:.5f}"


def test_parity_mode_c2_vs_reference_algorithm(L):
    """L4 at c2: the reference algorithm (fp64 sketches, per-tensor QM) on the device vs its
    NumPy restatement (pinned to the unmodified reference by tests/test_oracle_golden.py), at
    <= 1e-9 relative Frobenius."""
    cfg = CONFIGS["c2"]
    ta, tb = synth_pair(cfg)
    kw = dict(rank=cfg["rank"], bits=(8, 8, 8), power_iters=cfg["power_iters"], oversample=cfg["oversample"], seed=0)
    d, status, _ = L.lramm_device(ta, tb, L.LrammParams(**kw))
    torch.cuda.synchronize()
    assert int(status.item()) == 0
    ref = O.lramm(ta.cpu().numpy(), tb.cpu().numpy(), O.OracleParams(**kw))
    assert rel_dev(d, torch.from_numpy(ref).to(d.device)) <= 1e-9


# ------------------------------------------------------------------ int32 accumulators, bit-exact


def _igemm(N, M, Nn, K, qa, lda, qb, ldb, packed=False):
    out = torch.empty((M, Nn), dtype=torch.int32, device=qb.device)
    e = N.Epilogue()
    e.out_dtype, e.out, e.ldo = N.I32, out.data_ptr(), Nn
    fn = N.LIB.lramm_igemm_i4 if packed else N.LIB.lramm_igemm
    stream = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    N.check(fn(M, Nn, K, ctypes.c_void_p(qa.data_ptr()), lda, ctypes.c_void_p(qb.data_ptr()), ldb, ctypes.byref(e), 1,
               stream))
    return out


def _sample_rows(M, rng, block=128):
    starts = sorted({0, M // 2 - block // 2, M - block} | set(int(s) for s in rng.integers(0, M - block, 2)))
    return np.concatenate([np.arange(s, s + block) for s in starts])


@pytest.mark.parametrize("case", ["c2_E3_two_ctas_per_sm", "c5_sketch_nfast", "c3_sketch_int4_nfast"])
def test_igemm_accumulators_bit_exact_at_config_shapes(case):
    from paper_2405_16917_b200 import _native as N

    M, Nn, K, packed = {
        "c2_E3_two_ctas_per_sm": (4096, 4096, 256, False),  # 32 x 16 = 512 CTAs > 148 SMs
        "c5_sketch_nfast": (131072, 1056, 8192, False),      # A 1 GiB int8: N-fastest raster
        "c3_sketch_int4_nfast": (8192, 544, 8192, True),     # packed int4 A (64 MiB unpacked)
    }[case]
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev)
    g.manual_seed(len(case) * 7919 + M)
    cap = 7 if packed else 127
    a = torch.randint(-cap, cap + 1, (M, K), generator=g, device=dev, dtype=torch.int8)
    b = torch.randint(-127, 128, (Nn, K), generator=g, device=dev, dtype=torch.int8)
    if packed:
        lo, hi = a[:, 0::2].to(torch.uint8) & 0xF, a[:, 1::2].to(torch.uint8) & 0xF
        qa = (lo | (hi << 4)).contiguous()
        assert qa.shape[1] % 16 == 0
        acc = _igemm(N, M, Nn, K, qa, qa.shape[1], b, K, packed=True)
        del qa
    else:
        acc = _igemm(N, M, Nn, K, a, K, b, K)
    torch.cuda.synchronize()
    rows = _sample_rows(M, np.random.default_rng(7))
    a_s = a[torch.from_numpy(rows).to(dev)].cpu().numpy().astype(np.float64)
    exact = (a_s @ b.cpu().numpy().astype(np.float64).T).astype(np.int64)  # K * 127^2 < 2^53: exact
    got = acc[torch.from_numpy(rows).to(dev)].cpu().numpy().astype(np.int64)
    assert np.array_equal(got, exact)
    # every column tile / every row tile touched: checksum of all accumulators against int64 sums
    col_sum = torch.zeros(Nn, dtype=torch.int64, device=dev)
    a_sum = torch.zeros(K, dtype=torch.int64, device=dev)
    for r0 in range(0, M, 8192):  # int32 partial sums are exact for 8192-row chunks
        col_sum += acc[r0:r0 + 8192].sum(dim=0, dtype=torch.int64)
        a_sum += a[r0:r0 + 8192].to(torch.int32).sum(dim=0).to(torch.int64)
    exact_col = (a_sum.double()[None, :] @ b.double().T).to(torch.int64)[0]  # |sums| < 2^53: exact
    assert torch.equal(col_sum, exact_col)
