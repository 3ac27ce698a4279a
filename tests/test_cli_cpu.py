"""CLI host logic against the reference CLI's own outputs (tests/golden/cli, made by
tests/golden/make_cli_golden.py from the unmodified reference): generators and LRMM / CSV
writers byte-identical, spec / file / parameter errors -> exit code 2 before any device work,
the MAC-model columns of `sweep` identical (model_only grid)."""

import csv
import io
import json
import os

import numpy as np
import pytest

from paper_2405_16917_b200 import cli, matio
from paper_2405_16917_b200.errors import FormatError

G = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "cli")


@pytest.mark.parametrize("args,name", [
    (["--rows", "40", "--cols", "32", "--dist", "uniform", "--seed", "7"], "gen_a.lrmm"),
    (["--rows", "32", "--cols", "36", "--dist", "normal", "--seed", "8"], "gen_b.lrmm"),
    (["--rows", "9", "--cols", "7", "--dist", "lowrank", "--rank", "3", "--noise", "0.05", "--seed", "2"],
     "gen_lowrank.csv"),
    (["--rows", "6", "--cols", "5", "--dist", "exponential", "--seed", "1"], "gen_exp.csv"),
    (["--rows", "6", "--cols", "5", "--dist", "binary", "--seed", "1"], "gen_bin.lrmm"),
])
def test_gen_bytes_match_reference(tmp_path, args, name):
    out = tmp_path / name
    assert cli.main(["gen", *args, "-o", str(out)]) == 0
    assert out.read_bytes() == open(os.path.join(G, name), "rb").read()


def test_lrmm_roundtrip_and_format_errors(tmp_path):
    a = matio.generate(5, 3, matio.NORMAL01, 11)
    p = tmp_path / "a.lrmm"
    matio.save_matrix(a, p)
    assert np.array_equal(matio.load_matrix(p), a)
    raw = p.read_bytes()
    (tmp_path / "magic.lrmm").write_bytes(b"XXXX" + raw[4:])
    (tmp_path / "short.lrmm").write_bytes(raw[:-8])
    (tmp_path / "tiny.lrmm").write_bytes(raw[:10])
    bad = np.frombuffer(raw[28:], dtype="<f8").copy()
    bad[2] = np.nan
    (tmp_path / "nan.lrmm").write_bytes(raw[:28] + bad.tobytes())
    offsets = {"magic.lrmm": 0, "tiny.lrmm": 10, "nan.lrmm": 28}
    for name in ("magic.lrmm", "short.lrmm", "tiny.lrmm", "nan.lrmm"):
        with pytest.raises(FormatError) as ei:
            matio.load_matrix(tmp_path / name)
        if name in offsets:
            assert ei.value.offset == offsets[name]
    c = tmp_path / "a.csv"
    matio.save_matrix_csv(a, c)
    assert np.array_equal(matio.load_matrix_csv(c), a)
    (tmp_path / "ragged.csv").write_text("1,2\n3\n")
    with pytest.raises(FormatError):
        matio.load_matrix_csv(tmp_path / "ragged.csv")


def test_usage_errors_exit_2(tmp_path, capsys):
    a = os.path.join(G, "gen_a.lrmm")
    b = os.path.join(G, "gen_b.lrmm")
    (tmp_path / "bad.lrmm").write_bytes(b"LRMM")
    assert cli.main(["mm", "-a", str(tmp_path / "bad.lrmm"), "-b", b, "--strategy", "exact"]) == 2
    assert cli.main(["mm", "-a", a, "-b", str(tmp_path / "missing.lrmm"), "--strategy", "exact"]) == 2
    assert cli.main(["gen", "--rows", "3", "--cols", "3", "--dist", "lowrank", "-o", str(tmp_path / "x")]) == 2
    assert cli.main(["gen", "--rows", "3", "--cols", "3"]) == 2  # no -o
    (tmp_path / "spec.json").write_text('{"dims": [[4, 4, 4]], "distributions": ["uniform"], "seeds": [0]}')
    assert cli.main(["sweep", "--spec", str(tmp_path / "spec.json")]) == 2  # missing ranks/bits
    (tmp_path / "spec2.json").write_text('{"dims": [[4, 4]], "distributions": ["uniform"], "seeds": [0], '
                                         '"ranks": [2], "bits": [[8, 8, 8]]}')
    assert cli.main(["sweep", "--spec", str(tmp_path / "spec2.json")]) == 2
    (tmp_path / "spec3.json").write_text("{not json")
    assert cli.main(["sweep", "--spec", str(tmp_path / "spec3.json")]) == 2
    err = capsys.readouterr().err
    assert "error:" in err


def test_sweep_model_columns_match_reference(tmp_path):
    spec = json.load(open(os.path.join(G, "sweep_spec.json")))
    spec["model_only"] = True
    p = tmp_path / "spec.json"
    p.write_text(json.dumps(spec))
    out = tmp_path / "sweep.csv"
    assert cli.main(["sweep", "--spec", str(p), "--format", "csv", "-o", str(out)]) == 0
    ours = list(csv.DictReader(io.StringIO(out.read_text())))
    ref = list(csv.DictReader(open(os.path.join(G, "sweep.csv"))))
    assert [r for r in ours[0]] == [r for r in ref[0]]  # same columns, same order
    assert len(ours) == len(ref)
    for o, r in zip(ours, ref):  # canonical row order and the MAC model, byte for byte
        for col in ("dist", "m", "n", "k", "r", "d1", "d2", "d3", "seed", "macs_total", "macs_baseline",
                    "speedup_model"):
            assert o[col] == r[col], col
        assert o["rel_error"] == "" and o["wall_ns"] == ""
