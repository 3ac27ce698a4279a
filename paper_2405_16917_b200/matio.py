"""Host-side matrix files and seeded test matrices for the CLI (the reference's
`matcore.generate` / `Distribution`, `matcore.py:40-126`, and the LRMM container / CSV
I/O, `matcore.py:251-326`).

These stay on the host ("LRMM I/O staying on host"): they are
NumPy byte and RNG plumbing around the device pipeline, restated so that files and
seeded inputs are byte-identical to the reference's (same NumPy Philox streams, same
little-endian container layout, same CSV `repr` formatting).
"""

from __future__ import annotations

import struct
from dataclasses import dataclass

import numpy as np

from .errors import FormatError, ParameterError, ShapeError

_KINDS = ("uniform", "normal", "exponential", "binary", "lowrank")
_DIST_TAG = {"uniform": 1, "normal": 2, "exponential": 3, "binary": 4, "lowrank": 5}  # matcore.py:86


@dataclass(frozen=True)
class Distribution:
    """Entry distribution of `generate` (matcore.py:47-80): uniform U[0,1), normal N(0,1),
    exponential (rate 1), binary {0,1}, or lowrank sum_i (1/i) u_i v_i^T (+ Gaussian noise)."""

    kind: str
    rank: int = 0
    noise_sigma: float = 0.0

    def __post_init__(self):
        if self.kind not in _KINDS:
            raise ParameterError(f"unknown distribution kind {self.kind!r}")
        if self.kind == "lowrank":
            if self.rank < 1:
                raise ParameterError("lowrank distribution needs rank >= 1")
            if self.noise_sigma < 0:
                raise ParameterError("noise_sigma must be >= 0")

    @classmethod
    def lowrank(cls, rank, noise_sigma=0.0):
        return cls("lowrank", rank=rank, noise_sigma=float(noise_sigma))

    def label(self):
        """CSV label without commas (matcore.py:75-79)."""
        if self.kind == "lowrank":
            return f"lowrank({self.rank};{self.noise_sigma!r})"
        return self.kind


UNIFORM01 = Distribution("uniform")
NORMAL01 = Distribution("normal")
EXPONENTIAL1 = Distribution("exponential")
BINARY01 = Distribution("binary")


def _rng(seed, *context):
    """Philox(SeedSequence([seed, *context])) keyed generator (matcore.py:89-92)."""
    entropy = [int(seed) & 0xFFFFFFFFFFFFFFFF] + [int(c) & 0xFFFFFFFFFFFFFFFF for c in context]
    return np.random.Generator(np.random.Philox(np.random.SeedSequence(entropy)))


def generate(rows, cols, dist, seed):
    """Seeded rows x cols float64 matrix (matcore.py:95-126), identical draws to the reference."""
    if rows < 1 or cols < 1:
        raise ShapeError(f"dimensions must be positive, got {rows}x{cols}")
    if not isinstance(dist, Distribution):
        raise ParameterError("dist must be a Distribution")
    g = _rng(seed, _DIST_TAG[dist.kind], rows, cols, dist.rank)
    if dist.kind == "uniform":
        a = g.random((rows, cols))
    elif dist.kind == "normal":
        a = g.standard_normal((rows, cols))
    elif dist.kind == "exponential":
        a = g.standard_exponential((rows, cols))
    elif dist.kind == "binary":
        a = g.integers(0, 2, size=(rows, cols)).astype(np.float64)
    else:
        if dist.rank > min(rows, cols):
            raise ParameterError(f"lowrank rank {dist.rank} exceeds min(rows, cols) = {min(rows, cols)}")
        u = np.linalg.qr(g.standard_normal((rows, dist.rank)))[0]
        v = np.linalg.qr(g.standard_normal((cols, dist.rank)))[0]
        a = (u * (1.0 / np.arange(1, dist.rank + 1))) @ v.T
        if dist.noise_sigma > 0:
            a = a + dist.noise_sigma * g.standard_normal((rows, cols))
    return np.ascontiguousarray(a)


# ------------------------------------------------------------------ LRMM container
MAGIC = b"LRMM"
VERSION = 1
DTYPE_F64 = 1
DTYPE_I32 = 2
_HEADER = struct.Struct("<4sIIQQ")  # magic, version, dtype code, rows, cols (matcore.py:251)


def as_matrix(a, name="matrix"):
    """C-contiguous float64 2-D array with positive dims (matcore.py:31-38)."""
    arr = np.asarray(a, dtype=np.float64)
    if arr.ndim != 2:
        raise ShapeError(f"{name} must be 2-D, got ndim={arr.ndim}")
    if arr.shape[0] < 1 or arr.shape[1] < 1:
        raise ShapeError(f"{name} must have positive dimensions, got {arr.shape}")
    return np.ascontiguousarray(arr)


def _read_container(path, expect_dtype):
    with open(path, "rb") as fh:
        raw = fh.read()
    if len(raw) < _HEADER.size:
        raise FormatError("file shorter than header", len(raw))
    magic, version, code, rows, cols = _HEADER.unpack_from(raw, 0)
    if magic != MAGIC:
        raise FormatError(f"bad magic {magic!r}", 0)
    if version != VERSION:
        raise FormatError(f"unsupported version {version}", 4)
    if code != expect_dtype:
        raise FormatError(f"dtype code {code}, expected {expect_dtype}", 8)
    if rows < 1 or cols < 1:
        raise FormatError(f"non-positive dims {rows}x{cols}", 12)
    need = rows * cols * (8 if code == DTYPE_F64 else 4)
    body = raw[_HEADER.size:]
    if len(body) < need:
        raise FormatError(f"payload truncated: need {need} bytes, have {len(body)}", _HEADER.size + len(body))
    return body[:need], rows, cols


def save_matrix(a, path):
    """LRMM container, float64 little-endian payload (matcore.py:286-290)."""
    a = as_matrix(a)
    with open(path, "wb") as fh:
        fh.write(_HEADER.pack(MAGIC, VERSION, DTYPE_F64, a.shape[0], a.shape[1]))
        fh.write(a.astype("<f8", copy=False).tobytes())


def load_matrix(path):
    """Read a float64 LRMM file; non-finite payloads are rejected (matcore.py:293-300)."""
    payload, rows, cols = _read_container(path, DTYPE_F64)
    a = np.frombuffer(payload, dtype="<f8").astype(np.float64).reshape(rows, cols)
    if not np.isfinite(a).all():
        raise FormatError("payload contains non-finite values", _HEADER.size)
    return np.ascontiguousarray(a)


def save_matrix_csv(a, path):
    """Headerless CSV, `repr` of each float (matcore.py:303-309)."""
    a = as_matrix(a)
    with open(path, "w") as fh:
        for row in a:
            fh.write(",".join(repr(x) for x in row.tolist()))
            fh.write("\n")


def load_matrix_csv(path):
    """Headerless CSV (matcore.py:312-326)."""
    rows = []
    with open(path) as fh:
        for lineno, line in enumerate(fh, 1):
            line = line.strip()
            if not line:
                continue
            try:
                rows.append([float(tok) for tok in line.split(",")])
            except ValueError as exc:
                raise FormatError(f"bad CSV value on line {lineno}: {exc}", 0) from None
    if not rows or any(len(r) != len(rows[0]) for r in rows):
        raise FormatError("empty or ragged CSV matrix", 0)
    return as_matrix(np.array(rows))


def load_any(path):
    return load_matrix_csv(path) if str(path).endswith(".csv") else load_matrix(path)


def save_any(a, path):
    if str(path).endswith(".csv"):
        save_matrix_csv(a, path)
    else:
        save_matrix(a, path)
