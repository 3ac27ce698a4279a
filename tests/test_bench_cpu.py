"""bench.py host logic without a GPU: BASELINE config shapes, the algorithmic-work models and the
per-stage roofline table built from a kernel-time dictionary."""

import json
import os

import bench

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_configs_match_baseline():
    base = json.load(open(os.path.join(ROOT, "BASELINE.json")))
    c = bench.CONFIGS
    assert "m=n=k=4096" in base["configs"][1] and (c["c2"]["m"], c["c2"]["k"], c["c2"]["n"]) == (4096,) * 3
    assert (c["c2"]["rank"], c["c2"]["oversample"], c["c2"]["power_iters"]) == (256, 16, 1)
    assert (c["c3"]["rank"], c["c3"]["oversample"], c["c3"]["power_iters"], c["c3"]["sketch_bits"]) == (512, 32, 2, 4)
    assert (c["c4"]["pairs"], c["c4"]["m"], c["c4"]["rank"], c["c4"]["oversample"]) == (64, 2048, 128, 10)
    assert (c["c5"]["m"], c["c5"]["k"], c["c5"]["n"], c["c5"]["rank"]) == (131072, 8192, 8192, 1024)
    assert bench.effective_ops(c["c2"]) == 2 * 4096 ** 3


def test_stage_rooflines_classify_and_bound():
    per = {
        "void lramm::jacobi_cluster_kernel<9, false>(JacobiArgs)": [2000.0 * 5, 10],
        "void lramm::igemm_tn_kernel<1, false, false>(...)": [150.0 * 5, 45],
        "void lramm::epilogue_kernel<false>(...)": [40.0 * 5, 45],
        "void lramm::quantize_tile_kernel<float, 1, 2, false, false>(...)": [40.0 * 5, 10],
        "void lramm::absmax_tile_kernel<float, 4, 6>(...)": [30.0 * 5, 10],
        "lramm::chol_tiles_kernel(...)": [500.0 * 5, 40],
        "void lramm::dgemm_kernel<true, true>(...)": [300.0 * 5, 40],
        "lramm::omega_kernel(...)": [0.0, 0],
        "Memset (Device)": [10.0 * 5, 100],
    }
    st = bench.stage_rooflines(per, 5, bench.CONFIGS["c2"], {"hbm_gbs": 6500.0})
    assert st["small_svd"]["us_per_step"] == 2000.0
    assert st["int8_gemm"]["us_per_step"] == 190.0
    assert st["quantize"]["us_per_step"] == 70.0
    assert st["fp64_qr"]["us_per_step"] == 800.0
    assert st["other"]["us_per_step"] == 10.0
    for k in ("quantize", "int8_gemm", "fp64_qr", "small_svd"):
        assert 0.0 < st[k]["frac"] and st[k]["roofline_us"] > 0.0
    assert st["quantize"]["bound"] == "hbm" and st["small_svd"]["bound"] == "fp64"
