"""Report path on the B200: evaluate / combined_bound / leading_sigmas / quantized_svd_approx."""
import numpy as np
import pytest

import lramm_oracle as O

pytestmark = pytest.mark.gpu


def test_evaluate_matches_host_measurement():
    from paper_2405_16917_b200 import LrammParams
    from paper_2405_16917_b200 import report as R

    a = O.synth(300, 260, "exp:20", 8, 0, 0)
    b = O.synth(260, 280, "exp:20", 8, 0, 1)
    p = LrammParams(rank=24, bits=(8, 8, 8), power_iters=1, oversample=8, seed=4)
    d, rep = R.evaluate(a, b, p)
    exact = a.astype(np.float64) @ b.astype(np.float64)
    assert rep.rel_error == pytest.approx(O.rel_fro(d, exact), rel=1e-10)
    assert rep.fro_error == pytest.approx(np.linalg.norm(d - exact), rel=1e-10)
    # bound from LAPACK singular values with the restated formula
    sa = np.linalg.svd(a.astype(np.float64), compute_uv=False)
    sb = np.linalg.svd(b.astype(np.float64), compute_uv=False)
    bi = R.BoundInputs(m=300, n=280, k=260, r=24, sigma1=sa[0], sigma_r1=sa[24], gamma1=sb[0], gamma_r1=sb[24],
                       d1=8, d2=8, d3=8, q=1)
    assert rep.bound_combined == pytest.approx(R.lramm_general_bound(bi), rel=1e-9)
    assert rep.sigma_source == "oracle"
    assert rep.rel_error * np.linalg.norm(exact) <= rep.bound_combined
    assert set(rep.to_dict()) >= {"fro_error", "rel_error", "bound_combined", "macs", "wall_ns"}


def test_leading_sigmas_sources():
    from paper_2405_16917_b200 import report as R

    a = O.synth(600, 520, "exp:30", 9, 0, 0).astype(np.float64)
    s, src = R.leading_sigmas(a, 10, seed=3)
    assert src == "rsvd"  # min dim 520 > the reference's oracle cap (matcore.py:23)
    ref = O.rsvd(a, 10, 1, 10, 3).sigma  # the reference's estimate: RsvdParams(rank, q=1, seed)
    assert np.max(np.abs(s - ref)) <= 1e-9 * ref[0]
    s2, src2 = R.leading_sigmas(a[:300], 10)
    assert src2 == "oracle"
    assert np.max(np.abs(s2 - np.linalg.svd(a[:300], compute_uv=False)[:10])) <= 1e-12


def test_quantized_svd_approx_matches_reference_algorithm():
    from paper_2405_16917_b200 import report as R

    a = O.synth(120, 90, "exp:10", 10, 0, 0).astype(np.float64)
    qu, qv, rec = R.quantized_svd_approx(a, 12, 8, 8)
    u, s, vt = np.linalg.svd(a, full_matrices=False)
    du, su = O.quantize_tensor(u[:, :12] * s[:12], 8)
    dv, sv = O.quantize_tensor(vt[:12].T, 8)
    ref = O.dequantize(du, su) @ O.dequantize(dv, sv).T
    assert qu.bits == 8 and qv.bits == 8 and qu.data.shape == (120, 12) and qv.data.shape == (90, 12)
    assert O.rel_fro(rec, ref) <= 1e-3
    with pytest.raises(R.ParameterError):
        R.quantized_svd_approx(a, 91, 8, 8)
