"""`mm` / `sweep` / `profile` through the CLI on the B200 against the reference CLI's outputs
on the same files (tests/golden/cli, from tests/golden/make_cli_golden.py)."""

import csv
import io
import json
import os

import numpy as np
import pytest

from paper_2405_16917_b200 import cli, matio

pytestmark = pytest.mark.gpu
G = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "cli")
A = os.path.join(G, "gen_a.lrmm")
B = os.path.join(G, "gen_b.lrmm")


def _rel(x, y):
    return float(np.linalg.norm(x - y) / np.linalg.norm(y))


def test_mm_qgemm_bitwise(tmp_path):
    out = tmp_path / "d.lrmm"
    assert cli.main(["mm", "-a", A, "-b", B, "--strategy", "qgemm", "--bits", "8", "-o", str(out)]) == 0
    assert out.read_bytes() == open(os.path.join(G, "mm_qgemm.lrmm"), "rb").read()


def test_mm_exact(tmp_path):
    out = tmp_path / "d.lrmm"
    assert cli.main(["mm", "-a", A, "-b", B, "--strategy", "exact", "-o", str(out)]) == 0
    assert _rel(matio.load_matrix(out), matio.load_matrix(os.path.join(G, "mm_exact.lrmm"))) < 1e-14


def test_mm_lramm_matches_reference(tmp_path, capsys):
    out = tmp_path / "d.lrmm"
    assert cli.main(["mm", "-a", A, "-b", B, "--strategy", "lramm", "--rank", "8", "--bits", "8,8,8",
                     "--power-iters", "1", "--oversample", "6", "--seed", "5", "-o", str(out)]) == 0
    rep = json.loads(capsys.readouterr().out)
    ref = json.load(open(os.path.join(G, "mm_lramm.json")))
    assert rep["macs"] == ref["macs"]
    assert set(rep["wall_ns"]) == set(ref["wall_ns"])
    assert _rel(matio.load_matrix(out), matio.load_matrix(os.path.join(G, "mm_lramm.lrmm"))) <= 1e-3


def test_mm_report_fields(tmp_path, capsys):
    assert cli.main(["mm", "-a", A, "-b", B, "--strategy", "lramm", "--rank", "8", "--preset", "balanced",
                     "--report"]) == 0
    rep = json.loads(capsys.readouterr().out)
    for key in ("rel_error", "fro_error", "bound_combined"):
        assert key in rep and np.isfinite(rep[key])
    assert cli.main(["mm", "-a", A, "-b", B, "--strategy", "qgemm", "--bits", "8", "--report",
                     "--format", "csv"]) == 0
    head, row = capsys.readouterr().out.strip().split("\n")
    assert head.split(",")[:5] == ["strategy", "m", "k", "n", "wall_ns"] and len(row.split(",")) == len(head.split(","))


def test_sweep_matches_reference(tmp_path):
    out = tmp_path / "sweep.csv"
    assert cli.main(["sweep", "--spec", os.path.join(G, "sweep_spec.json"), "--format", "csv", "--threads", "2",
                     "-o", str(out)]) == 0
    ours = list(csv.DictReader(io.StringIO(out.read_text())))
    ref = list(csv.DictReader(open(os.path.join(G, "sweep.csv"))))
    assert len(ours) == len(ref)
    for o, r in zip(ours, ref):
        for col in ("dist", "m", "n", "k", "r", "d1", "d2", "d3", "seed", "macs_total", "macs_baseline",
                    "speedup_model"):
            assert o[col] == r[col], col
        for col in ("rel_error_dq4", "rel_error_dq8", "bound"):  # bit-exact qgemm; exact product / sigmas fp64
            assert float(o[col]) == pytest.approx(float(r[col]), rel=1e-9), col
        # the chained per-tensor quantisers: within the reference's own backend spread
        assert abs(float(o["rel_error"]) - float(r["rel_error"])) <= 0.02 * float(r["rel_error"]) + 2e-3
        assert int(o["wall_ns"]) > 0


def test_profile_matches_reference_model(tmp_path):
    out = tmp_path / "p.json"
    assert cli.main(["profile", "--rows", "48", "--cols", "40", "--inner", "36", "--rank", "8", "--bits", "8,8,4",
                     "--seed", "2", "-o", str(out)]) == 0
    ours = json.load(open(out))
    ref = json.load(open(os.path.join(G, "profile.json")))
    for key in ("m", "n", "k", "r", "d1", "d2", "d3", "q", "seed", "macs", "mac_shares"):
        assert ours[key] == ref[key], key
    assert set(ours["wall_ns"]) == set(ref["wall_ns"]) and ours["wall_ns"]["total"] > 0
    assert sum(ours["wall_shares"].values()) == pytest.approx(1.0)
