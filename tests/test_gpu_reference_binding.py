"""The INTEGRATION.md section 1 stub, taken verbatim from the document, bound into the reference.

The reference picks its kernel backend in `lramm/_kernels/__init__.py:8-39`; INTEGRATION.md shows
the `_cuda.py` stub a maintainer would add over `liblramm_cuda.so`.  This module executes that
code block as written, installs its four functions as the reference's kernel plugin
(`oracle/_ref`: the unmodified reference built by `oracle/build_ref.sh`) and restates the
reference's own cross-backend tests (`pkg/tests/test_backends.py`, file:line in each docstring)
with the CUDA backend in place of the compiled one, then runs the reference's own
`quantize` / `qgemm` / `oracle_svd` / `lramm` code on top of it.  Skipped when the reference
install is absent.
"""

import os
import re
import sys
import types

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def ref():
    os.environ["LRAMM_PURE_PYTHON"] = "1"  # the NumPy backend is the comparison side
    path = os.path.join(ROOT, "oracle", "_ref")
    if path not in sys.path:
        sys.path.insert(0, path)
    try:
        import lramm
    except Exception as exc:  # pragma: no cover
        pytest.skip(f"reference install not present: {exc}")
    return lramm


@pytest.fixture(scope="module")
def stub():
    import paper_2405_16917_b200  # noqa: F401  (fails loudly when the library is missing)

    text = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    sec = text[text.index("## 1. Kernel-plugin level"):]
    code = re.search(r"```python\n(.*?)```", sec, re.S).group(1)
    assert "lramm_host_imatmul" in code and "def svd(a)" in code
    os.environ["LRAMM_CUDA_LIB"] = os.path.join(ROOT, "paper_2405_16917_b200", "liblramm_cuda.so")
    mod = types.ModuleType("lramm_cuda_stub")
    exec(compile(code, "INTEGRATION.md:_cuda.py", "exec"), mod.__dict__)
    return mod


@pytest.fixture()
def bound(ref, stub, monkeypatch):
    """The reference with the stub installed as its kernel plugin (what the three lines added to
    `_kernels/__init__.py` do at import time)."""
    k = ref._kernels
    for name in ("matmul", "imatmul", "scale_round_clip", "svd"):
        monkeypatch.setattr(k, name, getattr(stub, name))
    monkeypatch.setattr(k, "BACKEND", "cuda")
    assert ref.backend_name() == "cuda"
    return ref


def pure(ref):
    from lramm._kernels import _pure

    return _pure


def test_matmul_backends_agree(ref, stub):
    """test_backends.py:26-32"""
    a = ref.generate(37, 23, ref.NORMAL01, 1)
    b = ref.generate(23, 41, ref.NORMAL01, 2)
    want = pure(ref).matmul(a, b)
    assert np.max(np.abs(stub.matmul(a, b) - want)) <= 1e-12 * (np.max(np.abs(want)) + 1.0)
    with pytest.raises(ValueError):
        stub.matmul(a, a)


def test_imatmul_backends_identical(ref, stub):
    """test_backends.py:35-39"""
    rng = np.random.Generator(np.random.Philox(key=3))
    a = rng.integers(-127, 128, size=(19, 31)).astype(np.int32)
    b = rng.integers(-127, 128, size=(31, 11)).astype(np.int32)
    got = stub.imatmul(a, b)
    assert got.dtype == np.int64 and np.array_equal(got, pure(ref).imatmul(a, b))


def test_quantize_backends_identical(ref, stub):
    """test_backends.py:42-52"""
    a = ref.generate(29, 17, ref.UNIFORM01, 4) * 2.0 - 1.0
    assert np.array_equal(stub.scale_round_clip(a, 127.0, 127), pure(ref).scale_round_clip(a, 127.0, 127))
    halves = np.array([[0.5, 1.5, 2.5, -0.5, -1.5, -2.5]])
    assert np.array_equal(stub.scale_round_clip(halves, 1.0, 127), np.array([[0, 2, 2, 0, -2, -2]], dtype=np.int32))


@pytest.mark.parametrize("shape", [(20, 20), (35, 14), (14, 35)])
def test_svd_backends_agree_on_spectrum(ref, stub, shape):
    """test_backends.py:55-60"""
    a = ref.generate(*shape, ref.NORMAL01, 5)
    s_cuda = stub.svd(a)[1]
    s_lapack = pure(ref).svd(a)[1]
    assert np.max(np.abs(s_cuda - s_lapack)) <= 1e-10 * max(s_lapack[0], 1.0)


def test_svd_contracts(ref, stub):
    """test_backends.py:63-72"""
    a = ref.generate(33, 26, ref.UNIFORM01, 6)
    u, s, v = stub.svd(a)
    t = min(a.shape)
    assert u.shape == (33, t) and v.shape == (26, t)
    assert np.all(np.diff(s) <= 1e-12)
    assert np.linalg.norm(u.T @ u - np.eye(t)) <= 1e-8 * np.sqrt(t)
    assert np.linalg.norm(v.T @ v - np.eye(t)) <= 1e-8 * np.sqrt(t)
    assert np.linalg.norm(a - (u * s) @ v.T) <= 1e-10 * np.linalg.norm(a)


def test_reference_suite_smoke_on_cuda_backend(bound):
    """test_backends.py:85-103, the same contracts with the CUDA plugin active."""
    lr = bound
    a = lr.generate(40, 40, lr.UNIFORM01, 1)
    b = lr.generate(40, 40, lr.UNIFORM01, 2)
    f = lr.oracle_svd(a)
    assert lr.frobenius_norm(a - f.reconstruct()) <= 1e-10 * lr.frobenius_norm(a)
    d, _ = lr.lramm(a, b, lr.LrammParams(rank=6, bits=(8, 8, 4), seed=3))
    assert lr.relative_error(d, lr.gemm(a, b)) < 1.0
    q = lr.quantize(a, 8)
    assert np.max(np.abs(lr.dequantize(q) - a)) <= 0.5 / q.scale + 1e-15


@pytest.mark.parametrize("bits", [(16, 16, 16), (8, 8, 8), (24, 12, 4)])
def test_reference_pipeline_same_output_on_both_backends(ref, stub, monkeypatch, bits):
    """The reference's own `lramm()` (pipeline.py:159-214), once on its NumPy backend and once on
    the CUDA plugin: the quantised integers and integer products are bit-identical by
    construction, so the outputs can differ only through the SVD backends' rounding."""
    a = ref.generate(96, 80, ref.Distribution.lowrank(12, 1e-3), 11)
    b = ref.generate(80, 72, ref.Distribution.lowrank(12, 1e-3), 12)
    p = ref.LrammParams(rank=10, bits=bits, power_iters=1, seed=5)
    want, _ = ref.lramm(a, b, p)
    qa = ref.quantize(a, bits[0])
    k = ref._kernels
    for name in ("matmul", "imatmul", "scale_round_clip", "svd"):
        monkeypatch.setattr(k, name, getattr(stub, name))
    got, _ = ref.lramm(a, b, p)
    qa_cuda = ref.quantize(a, bits[0])
    assert np.array_equal(qa.data, qa_cuda.data) and qa.scale == qa_cuda.scale
    monkeypatch.undo()
    want_q = ref.qgemm(a, b, bits[0], bits[0])
    for name in ("matmul", "imatmul", "scale_round_clip", "svd"):
        monkeypatch.setattr(k, name, getattr(stub, name))
    assert np.array_equal(ref.qgemm(a, b, bits[0], bits[0]), want_q)
    rel = np.linalg.norm(got - want) / np.linalg.norm(want)
    # wide budgets: the chained quantisers sit far from their rounding boundaries (<= 1e-9, the L4
    # gate); at 8 / 4 bits a boundary flip is allowed up to the reference's own backend spread
    # (its compiled and NumPy backends differ by up to 1.85e-3)
    assert rel <= (1e-9 if min(bits) >= 16 else 2e-3), rel
