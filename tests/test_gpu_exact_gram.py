"""Exact integer Gram of tall per-tensor sketches (pipeline.cu gram_limbs_kernel):
the CholeskyQR of Y = X.Omega takes G = Y_int^T Y_int / S^2 from int8 limb products instead of an
fp64 GEMM.  The path is off by default; the row threshold is read once per process, so the
checks run in a subprocess with LRAMM_EXACT_GRAM_ROWS set to reach test-sized shapes; the fast-mode result must meet the L5
gate against the CPU restatement (the same algorithm with an fp64 Gram) and agree with the
fp64-Gram run of this package to far below it."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import os, sys
sys.path.insert(0, {root!r}); sys.path.insert(0, os.path.join({root!r}, "oracle"))
import numpy as np, torch
import lramm_oracle as O
import paper_2405_16917_b200 as L
m, k, n, r, p, q = {shape}
a = O.synth(m, k, "exp:32", 7, 0, 0)
b = O.synth(k, n, "exp:32", 7, 0, 1)
kw = dict(rank=r, bits=(8, 8, 8), power_iters=q, oversample=p, seed=3)
spec = dict(mode="fast", sketch_bits=8, power_bits=8, proj_bits=8, granularity="tensor")
d, _ = L.lramm(a, b, L.LrammParams(**kw, **spec))
ref = O.lramm(a, b, O.OracleParams(**kw, spec=O.SketchSpec(8, 8, 8, "tensor")))
np.save({out!r}, d)
print("REL", float(np.linalg.norm(d - ref) / np.linalg.norm(ref)))
"""


def _run(shape, rows_thr, out):
    env = dict(os.environ, LRAMM_EXACT_GRAM_ROWS=str(rows_thr))
    src = SCRIPT.format(root=ROOT, shape=shape, out=out)
    r = subprocess.run([sys.executable, "-c", src], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    return float([l for l in r.stdout.splitlines() if l.startswith("REL")][-1].split()[1])


@pytest.mark.parametrize("shape", [(4096, 1024, 768, 64, 10, 1), (6000, 700, 900, 48, 8, 0)])
def test_exact_gram_sketch_matches_restatement(tmp_path, shape):
    import numpy as np

    rel_exact = _run(shape, 1024, str(tmp_path / "exact.npy"))  # tall sketches take the exact Gram
    rel_fp64 = _run(shape, 0, str(tmp_path / "fp64.npy"))       # path off: the fp64 DMMA Gram
    assert rel_exact <= 1e-3 and rel_fp64 <= 1e-3
    d1, d2 = np.load(tmp_path / "exact.npy"), np.load(tmp_path / "fp64.npy")
    assert np.linalg.norm(d1 - d2) <= 1e-6 * np.linalg.norm(d2)
