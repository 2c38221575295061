"""B200-native (sm_100a) HoSZp hot path -- drop-in for the reference package
``hoszp`` 0.1.0 (arxiv 2408.11971) on its data-parallel path: compress,
decompress, negate, scalar add / sub / multiply, mean, variance.

Same public names, argument meanings, errors and ``.hsz`` byte layout as the
reference (pkg/src/hoszp/__init__.py); the O(N) work runs in hand-written
CUDA kernels (``csrc/``) behind the C ABI of ``include/hsz_b200.h``.
"""

from .errors import (
    BadMagic,
    FormatError,
    GeometryMismatch,
    HoszpError,
    OutlierOverflow,
    ParamsMismatch,
    QuantOverflow,
    TruncatedStream,
    VerificationMismatch,
    VersionMismatch,
)
from .model import CompressedStream, QuantArray, QuantParams, deserialize, serialize
from .codec import (
    RawArray,
    compress,
    decode_to_quant,
    decompress,
    dequantize,
    encode_from_quant,
    quantize,
    read_raw,
    resolve_eps,
    write_raw,
)
from .device import DeviceStream
from .hszio import read_hsz, serialize_device, write_hsz
from .ops import (
    REDUCTIONS,
    STREAM_OPS,
    ScalarBin,
    apply_reduction,
    apply_stream_op,
    block_means,
    covariance,
    elementwise_add,
    elementwise_sub,
    hadamard,
    ssim_global,
    mean,
    negate,
    scalar_add,
    scalar_mul,
    scalar_sub,
    stddev,
    variance,
)

__version__ = "0.1.0+b200"
