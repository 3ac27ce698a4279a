"""CLI goldens from the UNMODIFIED reference CLI (test infrastructure).

    python tests/golden/make_cli_golden.py        # needs oracle/_ref (oracle/build_ref.sh)

Runs `python -m lramm.cli` from `oracle/_ref` and writes, under tests/golden/cli/:
  gen_*.lrmm / gen_*.csv   `lramm gen` outputs (seeded generators + LRMM / CSV writers)
  mm_lramm.lrmm, mm_lramm.json, mm_qgemm.lrmm, mm_exact.lrmm   `lramm mm` on gen_* inputs
  sweep.csv, sweep_spec.json                                  `lramm sweep` (small grid)
  profile.json                                                `lramm profile`
"""

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
OUT = os.path.join(HERE, "cli")
ENV = dict(os.environ, PYTHONPATH=os.path.join(ROOT, "oracle", "_ref"))

SPEC = """{
  "dims": [[24, 20, 16], [18, 12, 30]],
  "distributions": ["uniform", {"kind": "lowrank", "rank": 6, "noise_sigma": 0.01}],
  "seeds": [0, 3],
  "ranks": [4],
  "bits": [[8, 8, 8], [8, 8, 4]],
  "power_iters": 1,
  "oversample": 4
}
"""


def ref(*args, stdout=None):
    r = subprocess.run([sys.executable, "-m", "lramm.cli", *args], env=ENV, cwd=OUT, capture_output=True, text=True)
    if r.returncode != 0:
        raise SystemExit(f"reference CLI failed: {args}\n{r.stderr}")
    if stdout:
        with open(os.path.join(OUT, stdout), "w") as fh:
            fh.write(r.stdout)


def main():
    os.makedirs(OUT, exist_ok=True)
    ref("gen", "--rows", "40", "--cols", "32", "--dist", "uniform", "--seed", "7", "-o", "gen_a.lrmm")
    ref("gen", "--rows", "32", "--cols", "36", "--dist", "normal", "--seed", "8", "-o", "gen_b.lrmm")
    ref("gen", "--rows", "9", "--cols", "7", "--dist", "lowrank", "--rank", "3", "--noise", "0.05", "--seed", "2",
        "-o", "gen_lowrank.csv")
    ref("gen", "--rows", "6", "--cols", "5", "--dist", "exponential", "--seed", "1", "-o", "gen_exp.csv")
    ref("gen", "--rows", "6", "--cols", "5", "--dist", "binary", "--seed", "1", "-o", "gen_bin.lrmm")
    ref("mm", "-a", "gen_a.lrmm", "-b", "gen_b.lrmm", "--strategy", "lramm", "--rank", "8", "--bits", "8,8,8",
        "--power-iters", "1", "--oversample", "6", "--seed", "5", "-o", "mm_lramm.lrmm", stdout="mm_lramm.json")
    ref("mm", "-a", "gen_a.lrmm", "-b", "gen_b.lrmm", "--strategy", "qgemm", "--bits", "8", "-o", "mm_qgemm.lrmm")
    ref("mm", "-a", "gen_a.lrmm", "-b", "gen_b.lrmm", "--strategy", "exact", "-o", "mm_exact.lrmm")
    with open(os.path.join(OUT, "sweep_spec.json"), "w") as fh:
        fh.write(SPEC)
    ref("sweep", "--spec", "sweep_spec.json", "--format", "csv", "-o", "sweep.csv")
    ref("profile", "--rows", "48", "--cols", "40", "--inner", "36", "--rank", "8", "--bits", "8,8,4",
        "--seed", "2", "-o", "profile.json")


if __name__ == "__main__":
    main()
