"""CPU-side checks of the C-ABI boundary: the library loads, exports every symbol the
header declares, and the host-side mirror of the reference surface validates like
the reference (no compute: there is no GPU in the build container)."""

import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "lramm_cuda.h")
LIB = os.path.join(ROOT, "paper_2405_16917_b200", "liblramm_cuda.so")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(lramm_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(LIB)
    names = declared_symbols()
    assert len(names) >= 20
    for name in names:
        assert hasattr(lib, name), name


def test_binding_signatures_cover_header():
    from paper_2405_16917_b200 import _native

    assert sorted(_native.SIGNATURES) == declared_symbols()


def test_version_and_device_check_without_gpu():
    from paper_2405_16917_b200 import _native as N

    assert b"sm_100a" in N.LIB.lramm_version()
    rc = N.LIB.lramm_device_check()
    assert rc in (N.OK, N.ERR_UNSUPPORTED)


def test_struct_layouts_match_header():
    from paper_2405_16917_b200 import _native as N

    assert ctypes.sizeof(N.Params) == 64
    assert N.Params.alpha.offset == 24 and N.Params.mode.offset == 40
    assert ctypes.sizeof(N.Epilogue) == 96
    assert ctypes.sizeof(N.Timings) == 20
    # lramm_comm_t: two communicators, rank/world/flags/reserved, two function pointers
    assert ctypes.sizeof(N.Comm) == 48
    assert N.Comm.rank.offset == 16 and N.Comm.all_reduce.offset == 32 and N.Comm.all_gather.offset == 40


def test_params_validation_mirrors_reference():
    import paper_2405_16917_b200 as L

    with pytest.raises(L.ParameterError):
        L.LrammParams(rank=1)
    with pytest.raises(L.ParameterError):
        L.LrammParams(rank=4, bits=(8, 8))
    with pytest.raises(L.ParameterError):
        L.LrammParams(rank=4, bits=(8, 8, 99))
    with pytest.raises(L.ParameterError):
        L.LrammParams(rank=4, power_iters=-1)
    with pytest.raises(L.ParameterError):
        L.RsvdParams(rank=0)
    assert L.preset("balanced")["bits"] == (8, 8, 4)
    with pytest.raises(L.ParameterError):
        L.preset("nope")


def test_shape_errors_raise_before_device():
    import paper_2405_16917_b200 as L

    a = np.ones((8, 8))
    with pytest.raises(L.ShapeError):
        L.lramm(a, np.ones((9, 4)), L.LrammParams(rank=2))
    with pytest.raises(L.ParameterError):
        L.lramm(a, a, L.LrammParams(rank=20))
    with pytest.raises(L.ShapeError):
        L.lramm(a, a, L.LrammParams(rank=2), c=np.ones((3, 3)))
    with pytest.raises(L.ParameterError):
        L.lramm(a, a, L.LrammParams(rank=2, bits=(25, 8, 8)))


def test_oracle_svd_size_cap_is_the_references():
    """matcore.py:23, :240-243 and test_matcore.py:241: min dim > 512 raises OracleLimitError before
    any device work; the cap is a module constant read at call time, so a harness can raise it
     -- without a GPU the raised cap then reaches the no-fallback error instead."""
    import sys

    import paper_2405_16917_b200 as L

    rsvd = sys.modules["paper_2405_16917_b200.rsvd"]  # the package re-exports the rsvd function under this name
    assert rsvd.ORACLE_MAX_MIN_DIM == 512
    with pytest.raises(L.OracleLimitError):
        L.oracle_svd(np.zeros((513, 600)))
    with pytest.raises(L.OracleLimitError):
        L.oracle_svd(np.zeros((4096, 544)))
    assert issubclass(L.OracleLimitError, ValueError)  # errors.py:16 hierarchy


def test_no_cpu_fallback_without_device():
    import torch

    import paper_2405_16917_b200 as L

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        L.lramm(np.ones((8, 8)), np.ones((8, 8)), L.LrammParams(rank=2))


def test_cost_model_matches_oracle():
    import lramm_oracle as O

    import paper_2405_16917_b200 as L

    cm = L.cost_model(4096, 4096, 4096, 256, 64, 8, 8, 8)
    ref = O.cost_model(4096, 4096, 4096, 256, 64, 8, 8, 8)
    for s in L.STAGES + ("baseline_qgemm", "exact_gemm"):
        assert getattr(cm, s) == ref[s]


def test_child_seeds_match_oracle():
    import lramm_oracle as O

    from paper_2405_16917_b200.pipeline import _child_seeds

    for s in (0, 1, 12345, 2**63):
        assert _child_seeds(s) == O.child_seeds(s)


def test_omega_key_and_ziggurat_tables_reproduce_numpy():
    """The device Omega generator's inputs: the Philox key from SeedSequence, and the ziggurat
    tables in csrc/ziggurat_tables.h, replayed by a scalar model of the draw against NumPy."""
    import math
    import os
    import re

    import lramm_oracle as O  # noqa: F401

    from paper_2405_16917_b200._device import OmegaCache

    k0, k1 = OmegaCache.philox_key(77, 40, 9)
    st = np.random.Philox(np.random.SeedSequence([77, 0x534B, 40, 9])).state["state"]
    assert (k0, k1) == (int(st["key"][0]), int(st["key"][1])) and not st["counter"].any()
    hdr = open(os.path.join(os.path.dirname(__file__), "..", "paper_2405_16917_b200", "csrc",
                            "ziggurat_tables.h")).read()

    def table(name):
        body = re.search(name + r"\[256\] = \{(.*?)\};", hdr, re.S).group(1)
        return [float(v) if "." in v or "e" in v else int(v.replace("ULL", "")) for v in
                [t.strip() for t in body.split(",") if t.strip()]]

    K, W, F = table("kZigKHost"), table("kZigWHost"), table("kZigFHost")
    R = float(re.search(r"kZigR = ([0-9.e+-]+);", hdr).group(1))
    raw = np.random.Philox(np.random.SeedSequence([77, 0x534B, 40, 9])).random_raw(60000)
    u = lambda v: (int(v) >> 11) * (1.0 / 9007199254740992.0)  # noqa: E731
    out, i = [], 0
    while len(out) < 40000:
        r = int(raw[i]); i += 1
        idx, r = r & 0xFF, r >> 8
        sign, rabs = r & 1, (r >> 1) & 0x000FFFFFFFFFFFFF
        x = -rabs * W[idx] if sign else rabs * W[idx]
        if rabs < K[idx]:
            out.append(x)
        elif idx == 0:
            while True:
                xx, yy = -(1.0 / R) * math.log1p(-u(raw[i])), -math.log1p(-u(raw[i + 1]))
                i += 2
                if yy + yy > xx * xx:
                    out.append(-(R + xx) if (rabs >> 8) & 1 else R + xx)
                    break
        elif (F[idx - 1] - F[idx]) * u(raw[i]) + F[idx] < math.exp(-0.5 * x * x):
            i += 1
            out.append(x)
        else:
            i += 1
    ref = np.random.Generator(np.random.Philox(np.random.SeedSequence([77, 0x534B, 40, 9]))).standard_normal(40000)
    assert np.array_equal(np.array(out), ref)
    assert np.array_equal(O.gaussian_sketch(77, 40, 9).ravel(), ref[:360])  # the oracle's Omega is this stream


def test_shard_bounds_match_the_python_split():
    """lramm_shard_bounds (the C ABI's balanced contiguous split) == sharded.shard_bounds."""
    from paper_2405_16917_b200 import _native as N
    from paper_2405_16917_b200.sharded import _row_split

    for total in (1, 7, 8, 449, 8192, 131072):
        for world in (1, 2, 3, 4, 8):
            offs = _row_split(total, world)
            for rank in range(world):
                lo, hi = ctypes.c_int64(), ctypes.c_int64()
                N.LIB.lramm_shard_bounds(total, world, rank, ctypes.byref(lo), ctypes.byref(hi))
                assert (lo.value, hi.value) == (offs[rank], offs[rank + 1])


def test_sharded_entry_validates_before_touching_the_device():
    from paper_2405_16917_b200 import _native as N
    from paper_2405_16917_b200.pipeline import LrammParams, _params

    p = _params(LrammParams(rank=8))
    args = lambda comm: (None, None, N.F64, 64, 64, 64, ctypes.byref(p), None, None, None, N.F64, None, N.F64,  # noqa: E731
                         None, None, 0, comm, None)
    assert N.LIB.lramm_lramm_sharded(*args(None)) == N.ERR_PARAM
    comm = N.Comm()
    comm.rank, comm.world = 2, 2  # rank out of range
    assert N.LIB.lramm_lramm_sharded(*args(ctypes.byref(comm))) == N.ERR_PARAM
    comm.rank, comm.world = 0, 2  # live communicator without entry points
    assert N.LIB.lramm_lramm_sharded(*args(ctypes.byref(comm))) == N.ERR_PARAM
    assert b"all_reduce" in N.LIB.lramm_last_error()
    wide = _params(LrammParams(rank=8, bits=(16, 8, 8)))
    one = N.Comm()
    one.rank, one.world = 0, 1
    a = list(args(ctypes.byref(one)))
    a[6] = ctypes.byref(wide)
    assert N.LIB.lramm_lramm_sharded(*a) == N.ERR_UNSUPPORTED
    assert N.LIB.lramm_lramm_sharded_ws(4096, 4096, 4096, ctypes.byref(p), 2, 0) < \
        N.LIB.lramm_lramm_ws(4096, 4096, 4096, ctypes.byref(p))
