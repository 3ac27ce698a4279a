"""Case tables of the reference-generated goldens (shared by tests/golden/make_golden.py and the
tests; importing this module does not import the reference)."""

# Small lramm() cases: (name, m, k, n, input kind, rank, oversample, q, bits, seed)
LRAMM_CASES = [
    ("exp_q0_888", 96, 80, 72, "exp:8", 12, 6, 0, (8, 8, 8), 1),
    ("exp_q1_888", 96, 80, 72, "exp:8", 12, 6, 1, (8, 8, 8), 2),
    ("exp_q0_884", 96, 80, 72, "exp:8", 12, 6, 0, (8, 8, 4), 3),
    ("exp_q1_848", 128, 64, 96, "exp:12", 16, 10, 1, (8, 4, 8), 4),
    ("exp_q2_444", 64, 64, 64, "exp:6", 8, 4, 2, (4, 4, 4), 5),
    ("poly_q1_888", 120, 100, 110, "poly:1.5", 20, 8, 1, (8, 8, 8), 6),
    ("ragged_q0_886", 37, 53, 29, "exp:5", 5, 10, 0, (8, 8, 6), 7),
    ("clip_q1_888", 24, 40, 18, "exp:4", 10, 50, 1, (8, 8, 8), 8),  # oversample clipped
]
# lowrank / rank-deficient inputs (matcore.generate 'lowrank', matcore.py:115-125)
LOWRANK_CASES = [
    ("lowrank1_r2", 50, 50, 50, 1, 2, 10, 0, (8, 8, 8), 3),
    ("lowrank6_r6", 40, 40, 40, 6, 6, 10, 1, (8, 8, 8), 6),
]
