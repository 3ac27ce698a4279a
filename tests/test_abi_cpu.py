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


def test_omega_matches_reference_generator():
    import lramm_oracle as O

    from paper_2405_16917_b200._device import OMEGA

    om = OMEGA.host_omega(77, 40, 9)
    assert np.array_equal(om, O.gaussian_sketch(77, 40, 9))
