"""Golden values of the reference's closed-form bounds (bounds.py), for tests/test_report_cpu.py.

Run in the build container after oracle/build_ref.sh installed the reference into oracle/_ref:
    python tests/golden/make_bounds_golden.py
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(ROOT, "oracle", "_ref"))
from lramm import bounds  # the unmodified reference

CASES = [
    dict(m=1024, n=1024, k=1024, r=64, sigma1=1.0, sigma_r1=0.13, gamma1=0.9, gamma_r1=0.11, d1=8, d2=8, d3=4, q=1),
    dict(m=4096, n=2048, k=512, r=32, sigma1=3.5, sigma_r1=0.01, gamma1=2.0, gamma_r1=0.2, d1=4, d2=8, d3=16, q=0,
         lambda1=12.0, lambda2=7.5),
    dict(m=100, n=80, k=60, r=5, sigma1=10.0, sigma_r1=10.0, gamma1=1.0, gamma_r1=0.0, d1=24, d2=2, d3=3, q=2,
         lambda1=1.0, lambda2=2.0),
]
out = []
for c in CASES:
    bi = bounds.BoundInputs(**c)
    row = {"inputs": c, "lramm_general_bound": bounds.lramm_general_bound(bi), "qsvd_bound": bounds.qsvd_bound(bi)}
    if c.get("lambda1"):
        row["qgemm_bound"] = bounds.qgemm_bound(bi)
    out.append(row)
scalars = {
    "quant_scalar_var_bound": [bounds.quant_scalar_var_bound(3.0, 8), bounds.quant_scalar_var_bound(0.5, 2)],
    "quant_matrix_bound": [bounds.quant_matrix_bound(30, 40, 2.5)],
    "svd_trunc_bound": [bounds.svd_trunc_bound(0.3, 74, 64)],
    "rsvd_error_bound": [bounds.rsvd_error_bound(0.3, 10, 64, 1), bounds.rsvd_error_bound(0.01, 32, 512, 2)],
    "lramm_specific_bound": [bounds.lramm_specific_bound(1024, 64, 1.0, 0.05, 127, 127, 7)],
    "spectrum_shape_factor": [bounds.spectrum_shape_factor(1.0, 0.13, 1024, 64)],
}
with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "bounds_golden.json"), "w") as f:
    json.dump({"cases": out, "scalars": scalars}, f, indent=1)
print("wrote bounds_golden.json")
