"""B200-native LRAMM approximate matrix multiply (arXiv 2405.16917, Algorithm 3).

Drop-in for the hot path of the reference package `lramm`
(`pkg/src/lramm/__init__.py:6-76`): the same names for the pipeline, the
randomised SVD, the quantiser and quantised GEMM, the parameter/timing
dataclasses and the error types, computed by hand-written sm_100a CUDA
(liblramm_cuda.so, C ABI in include/lramm_cuda.h), plus the report path
(`evaluate`, the closed-form bounds, `quantized_svd_approx`), and the CLI front end
(`cli.py`: gen / mm / sweep / spectrum / profile, LRMM and CSV files and the seeded
generators on the host in `matio.py`).
"""

import os as _os

# Every product runs on several streams (two rsvd chains, helper and copy streams) and concurrent
# products multiply that; the default 8 hardware work queues make unrelated streams share a queue
# and serialise.  Only effective when set before the process creates its CUDA context.
_os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

from . import _native  # noqa: E402,F401  (fails loudly if liblramm_cuda.so is missing)
from .errors import (
    DegenerateDenominatorError,
    FormatError,
    LrammError,
    OracleLimitError,
    OverflowRiskError,
    ParameterError,
    ShapeError,
    UnsupportedError,
)
from .kernels import backend_name
from .pipeline import (
    STAGES,
    CostModel,
    LrammParams,
    StageTimings,
    cost_model,
    gemm,
    lramm,
    lramm_device,
    preset,
)
from .quant import (
    QuantizedMatrix,
    bit_cap,
    dequantize,
    integer_matmul,
    qgemm,
    quantize,
)
from .report import (
    BoundInputs,
    ErrorReport,
    combined_bound,
    evaluate,
    frobenius_norm,
    leading_sigmas,
    lramm_general_bound,
    lramm_specific_bound,
    qgemm_bound,
    qsvd_bound,
    quant_matrix_bound,
    quant_scalar_var_bound,
    quantized_svd_approx,
    relative_error,
    rsvd_error_bound,
    spectrum_shape_factor,
    svd_trunc_bound,
)
from .rsvd import (
    RsvdParams,
    SvdFactors,
    oracle_svd,
    range_finder,
    rsvd,
    truncate_svd,
)

__version__ = "0.1.0"
