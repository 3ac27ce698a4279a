"""ctypes binding of liblramm_cuda.so (include/lramm_cuda.h).

The product path has no CPU fallback: if the library is missing this module
raises at import, and every compute call fails loudly when no sm_100 device is
present.
"""

from __future__ import annotations

import ctypes
import os

from .errors import (
    LrammError,
    OverflowRiskError,
    ParameterError,
    ShapeError,
    UnsupportedError,
)

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "liblramm_cuda.so")

# lramm_status
OK, ERR_SHAPE, ERR_PARAM, ERR_OVERFLOW, ERR_NONCONV, ERR_UNSUPPORTED, ERR_CUDA, ERR_NONFINITE, ERR_WS = range(9)
# lramm_dtype / granularity / mode
F32, F64, I8, I32, I64, I4 = range(6)
GRAN_TENSOR, GRAN_ROW, GRAN_COL = range(3)
MODE_PARITY, MODE_FAST = range(2)


class NativeLibraryMissing(ImportError):
    pass


class Params(ctypes.Structure):
    _fields_ = [
        ("rank", ctypes.c_int32),
        ("oversample", ctypes.c_int32),
        ("power_iters", ctypes.c_int32),
        ("bits", ctypes.c_int32 * 3),
        ("alpha", ctypes.c_double),
        ("beta", ctypes.c_double),
        ("mode", ctypes.c_int32),
        ("sketch_bits", ctypes.c_int32),
        ("power_bits", ctypes.c_int32),
        ("proj_bits", ctypes.c_int32),
        ("granularity", ctypes.c_int32),
        ("reserved", ctypes.c_int32),
    ]


class Timings(ctypes.Structure):
    _fields_ = [(n, ctypes.c_float) for n in ("rsvd_ms", "scaling_ms", "gemm1_ms", "gemm2_ms", "gemm3_ms")]


class Epilogue(ctypes.Structure):
    _fields_ = [
        ("out_dtype", ctypes.c_int32),
        ("accumulate", ctypes.c_int32),
        ("transpose_out", ctypes.c_int32),
        ("c_dtype", ctypes.c_int32),
        ("out", ctypes.c_void_p),
        ("ldo", ctypes.c_int64),
        ("row_scale", ctypes.c_void_p),
        ("row_scale_inc", ctypes.c_int64),
        ("col_scale", ctypes.c_void_p),
        ("col_scale_inc", ctypes.c_int64),
        ("alpha", ctypes.c_double),
        ("beta", ctypes.c_double),
        ("c", ctypes.c_void_p),
        ("ldc", ctypes.c_int64),
    ]


# lramm_comm_t: collective entry points with NCCL's own signatures (include/lramm_cuda.h)
ALL_REDUCE_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int,
                                 ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p)
ALL_GATHER_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int,
                                 ctypes.c_void_p, ctypes.c_void_p)
COMM_FORCE = 1


class Comm(ctypes.Structure):
    _fields_ = [
        ("comm", ctypes.c_void_p),
        ("comm_b", ctypes.c_void_p),
        ("rank", ctypes.c_int32),
        ("world", ctypes.c_int32),
        ("flags", ctypes.c_int32),
        ("reserved", ctypes.c_int32),
        ("all_reduce", ctypes.c_void_p),
        ("all_gather", ctypes.c_void_p),
    ]


_i64, _i32, _vp, _sz, _d = ctypes.c_int64, ctypes.c_int, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_double
_P = ctypes.POINTER

# name -> (restype, argtypes); the exported surface of include/lramm_cuda.h
SIGNATURES = {
    "lramm_last_error": (ctypes.c_char_p, []),
    "lramm_version": (ctypes.c_char_p, []),
    "lramm_device_check": (_i32, []),
    "lramm_quantize": (_i32, [_vp, _i32, _i64, _i64, _i64, _i32, _i32, _i32, _vp, _i32, _i64, _vp, _vp, _vp, _sz, _vp]),
    "lramm_quantize_ws": (_sz, [_i64, _i64]),
    "lramm_scale_round_clip": (_i32, [_vp, _i64, _i64, _i64, _d, _i32, _vp, _i64, _vp]),
    "lramm_absmax": (_i32, [_vp, _i32, _i64, _i64, _i64, _i32, _vp, _vp, _vp]),
    "lramm_quantize_pair": (_i32, [_vp, _i32, _i64, _i64, _i64, _i32, _i32, _vp, _i64, _vp, _i32, _i32, _vp, _i64, _vp,
                                   _vp, _vp, _sz, _vp]),
    "lramm_quantize_amax": (_i32, [_vp, _i32, _i64, _i64, _i64, _i32, _i32, _i32, _vp, _vp, _i32, _i64, _vp, _vp]),
    "lramm_cholqr_pass": (_i32, [_vp, _i64, _i64, _i64, _vp, _vp, _i64, _vp, _vp, _vp, _sz, _vp]),
    "lramm_cholqr_pass_ws": (_sz, [_i64, _i64]),
    "lramm_dequant": (_i32, [_vp, _i64, _i64, _i64, _P(Epilogue), _vp]),
    "lramm_igemm": (_i32, [_i64, _i64, _i64, _vp, _i64, _vp, _i64, _P(Epilogue), _i32, _vp]),
    "lramm_igemm_i4": (_i32, [_i64, _i64, _i64, _vp, _i64, _vp, _i64, _P(Epilogue), _i32, _vp]),
    "lramm_omega": (_i32, [ctypes.c_uint64, ctypes.c_uint64, _i64, _i64, _vp, _vp, _sz, _vp]),
    "lramm_omega_ws": (_sz, [_i64, _i64]),
    "lramm_split_limbs": (_i32, [_vp, _i64, _i64, _i64, _i32, _vp, _i64, _vp]),
    "lramm_igemm_limbs": (_i32, [_i64, _i64, _i64, _vp, _i64, _i64, _i32, _vp, _i64, _i64, _i32, _vp, _P(Epilogue),
                                 _vp]),
    "lramm_dgemm": (_i32, [_i32, _i64, _i64, _i64, _vp, _i64, _vp, _i64, _vp, _i64, _vp, _sz, _vp]),
    "lramm_dgemm_ws": (_sz, [_i32, _i64, _i64, _i64]),
    "lramm_qr": (_i32, [_vp, _i64, _i64, _i64, _vp, _i64, _vp, _vp, _sz, _vp]),
    "lramm_qr_ws": (_sz, [_i64, _i64]),
    "lramm_svd": (_i32, [_vp, _i64, _i64, _vp, _vp, _vp, _vp, _vp, _sz, _vp]),
    "lramm_svd_ws": (_sz, [_i64, _i64]),
    "lramm_rsvd": (_i32, [_vp, _i32, _i64, _i64, _P(Params), _vp, _vp, _vp, _vp, _vp, _vp, _sz, _vp]),
    "lramm_rsvd_ws": (_sz, [_i64, _i64, _P(Params)]),
    "lramm_lramm": (_i32, [_vp, _vp, _i32, _i64, _i64, _i64, _P(Params), _vp, _vp, _vp, _i32, _vp, _i32, _vp, _vp,
                           _sz, _P(Timings), _vp]),
    "lramm_lramm_ws": (_sz, [_i64, _i64, _i64, _P(Params)]),
    "lramm_shard_bounds": (None, [_i64, ctypes.c_int32, ctypes.c_int32, _P(_i64), _P(_i64)]),
    "lramm_lramm_sharded": (_i32, [_vp, _vp, _i32, _i64, _i64, _i64, _P(Params), _vp, _vp, _vp, _i32, _vp, _i32, _vp,
                                   _vp, _sz, _P(Comm), _vp]),
    "lramm_lramm_sharded_ws": (_sz, [_i64, _i64, _i64, _P(Params), ctypes.c_int32, ctypes.c_int32]),
    "lramm_host_matmul": (_i32, [_vp, _vp, _vp, _i64, _i64, _i64]),
    "lramm_host_imatmul": (_i32, [_vp, _vp, _vp, _i64, _i64, _i64]),
    "lramm_host_scale_round_clip": (_i32, [_vp, _i64, _i64, _d, _i32, _vp]),
    "lramm_host_svd": (_i32, [_vp, _i64, _i64, _vp, _vp, _vp]),
    "lramm_host_lramm": (_i32, [_vp, _vp, _i32, _i64, _i64, _i64, _P(Params), _vp, _vp, _vp, _i32, _vp, _i32,
                                _P(Timings)]),
}


def _load():
    if not os.path.exists(LIB_PATH):
        raise NativeLibraryMissing(
            f"{LIB_PATH} is missing: build it with `python paper_2405_16917_b200/build.py` "
            "(there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


LIB = _load()

_ERRORS = {
    ERR_SHAPE: ShapeError,
    ERR_PARAM: ParameterError,
    ERR_OVERFLOW: OverflowRiskError,
    ERR_NONCONV: RuntimeError,
    ERR_UNSUPPORTED: UnsupportedError,
    ERR_CUDA: RuntimeError,
    ERR_NONFINITE: ParameterError,
    ERR_WS: RuntimeError,
}


def check(rc: int) -> None:
    if rc == OK:
        return
    msg = LIB.lramm_last_error().decode(errors="replace")
    exc = _ERRORS.get(rc, LrammError)
    raise exc(msg)


def last_error() -> str:
    return LIB.lramm_last_error().decode(errors="replace")
