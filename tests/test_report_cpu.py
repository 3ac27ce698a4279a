"""Report-path bounds (bounds.py restated in paper_2405_16917_b200.report) vs the reference's values."""
import json
import math
import os

import pytest

from paper_2405_16917_b200 import report as R

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "bounds_golden.json")))


@pytest.mark.parametrize("i", range(len(GOLD["cases"])))
def test_product_bounds_match_reference(i):
    case = GOLD["cases"][i]
    bi = R.BoundInputs(**case["inputs"])
    assert R.lramm_general_bound(bi) == pytest.approx(case["lramm_general_bound"], rel=1e-14)
    assert R.qsvd_bound(bi) == pytest.approx(case["qsvd_bound"], rel=1e-14)
    if "qgemm_bound" in case:
        assert R.qgemm_bound(bi) == pytest.approx(case["qgemm_bound"], rel=1e-14)


def test_scalar_bounds_match_reference():
    s = GOLD["scalars"]
    assert R.quant_scalar_var_bound(3.0, 8) == pytest.approx(s["quant_scalar_var_bound"][0], rel=1e-15)
    assert R.quant_scalar_var_bound(0.5, 2) == pytest.approx(s["quant_scalar_var_bound"][1], rel=1e-15)
    assert R.quant_matrix_bound(30, 40, 2.5) == pytest.approx(s["quant_matrix_bound"][0], rel=1e-15)
    assert R.svd_trunc_bound(0.3, 74, 64) == pytest.approx(s["svd_trunc_bound"][0], rel=1e-15)
    assert R.rsvd_error_bound(0.3, 10, 64, 1) == pytest.approx(s["rsvd_error_bound"][0], rel=1e-15)
    assert R.rsvd_error_bound(0.01, 32, 512, 2) == pytest.approx(s["rsvd_error_bound"][1], rel=1e-15)
    assert R.lramm_specific_bound(1024, 64, 1.0, 0.05, 127, 127, 7) == pytest.approx(
        s["lramm_specific_bound"][0], rel=1e-15)
    assert R.spectrum_shape_factor(1.0, 0.13, 1024, 64) == pytest.approx(s["spectrum_shape_factor"][0], rel=1e-15)


def test_bound_validation_errors():
    with pytest.raises(R.ParameterError):
        R.BoundInputs(m=0, n=3)
    with pytest.raises(R.ParameterError):
        R.BoundInputs(m=3, n=3, sigma1=1.0, sigma_r1=2.0)
    with pytest.raises(R.ParameterError):
        R.svd_trunc_bound(0.1, 4, 4)
    with pytest.raises(R.ParameterError):
        R.rsvd_error_bound(0.1, 4, 1, 0)
    with pytest.raises(R.ParameterError):
        R.quant_matrix_bound(2, 2, 0.0)
    with pytest.raises(R.ParameterError):
        R.lramm_specific_bound(4, 2, 1.0, -1.0, 7, 7, 7)
    assert math.isfinite(R.lramm_general_bound(R.BoundInputs(m=4, n=4, k=4, r=2, sigma1=1.0, gamma1=1.0)))
