"""Exception classes of the hot path.

Same names and subclass relations as the reference's error module
(`pkg/src/hoszp/errors.py:4-45`) so that callers catching e.g.
``QuantOverflow`` keep working when they switch to this package.  The CUDA
kernels report failures through a device error word (bit flags, see
``include/hsz_b200.h``); :func:`raise_for_flags` maps that word onto these
classes in the order the reference pipeline would have hit them.
"""

from __future__ import annotations


class HoszpError(Exception):
    """Root of every error raised by the package."""


class QuantOverflow(HoszpError):
    """A bin (or an intermediate bin computation) leaves the signed 63-bit
    working range, usually because eps is too small for the data range."""


class OutlierOverflow(HoszpError):
    """A block's first bin does not fit the int32 outlier slot."""


class ParamsMismatch(HoszpError):
    """Operands of a bivariate operation carry different parameters."""


class FormatError(HoszpError):
    """Serialized bytes could not be parsed."""


class BadMagic(FormatError):
    """The bytes do not begin with ``HSZP``."""


class VersionMismatch(FormatError):
    """Unsupported stream format version."""


class TruncatedStream(FormatError):
    """The bytes end before all declared sections are complete."""


class GeometryMismatch(FormatError):
    """Header fields and section sizes disagree."""


class VerificationMismatch(HoszpError):
    """A homomorphic result disagrees with the traditional workflow."""


class DeviceTimeout(HoszpError, RuntimeError):
    """A device-side wait gave up (the encoders' look-back watchdog,
    HSZ_ERR_LOOKBACK_TIMEOUT): the operation's output is undefined.  Not a
    reference error class -- it replaces a GPU hang."""


class CapacityExceeded(HoszpError):
    """Internal: an output section outgrew its preallocated device buffer.

    Never escapes the public API -- the host retries with the exact size the
    kernel reported."""


# Device error-word bits (mirrors HSZ_ERR_* in include/hsz_b200.h).
ERR_NONFINITE = 1 << 0        # raw input holds NaN/Inf        -> ValueError
ERR_QUANT_OVERFLOW = 1 << 1   # |floor((x+eps)/2eps)| >= 2^63   -> QuantOverflow
ERR_QUANT_RESOLUTION = 1 << 2  # repair pass could not honour eps -> QuantOverflow
ERR_PREFIX_OVERFLOW = 1 << 3  # decoded prefix sum beyond 63 bits -> QuantOverflow
ERR_RESCALE_OVERFLOW = 1 << 4  # smul rescale |bin| >= 2^63       -> QuantOverflow
ERR_OUTLIER_OVERFLOW = 1 << 5  # outlier outside int32            -> OutlierOverflow
ERR_CAPACITY = 1 << 6         # output buffer too small (retry)
ERR_OUTPUT_NONFINITE = 1 << 7  # decoded value overflowed the dtype -> ValueError
ERR_BAD_WIDTH = 1 << 8        # width > 64 in a stream           -> GeometryMismatch
ERR_LOOKBACK_TIMEOUT = 1 << 9  # encoder look-back watchdog fired   -> DeviceTimeout


def raise_for_flags(flags: int, what: str = "") -> None:
    """Raise the exception the reference would raise for this error word.

    Precedence follows the reference's stage order: input validation, then
    quantization, then prefix decoding, then rescaling, then the int32 guard
    applied when the resulting stream object is built.
    """
    flags = int(flags)
    if not flags:
        return
    tag = f" ({what})" if what else ""
    if flags & ERR_LOOKBACK_TIMEOUT:
        raise DeviceTimeout("an encoder's look-back wait timed out; the output is undefined "
                            "and the workspace was re-initialised" + tag)
    if flags & ERR_NONFINITE:
        raise ValueError("raw data must be finite (no NaN/Inf)" + tag)
    if flags & ERR_BAD_WIDTH:
        raise GeometryMismatch("width exceeds 64 bits" + tag)
    if flags & ERR_QUANT_OVERFLOW:
        raise QuantOverflow("quantization bin exceeds 63-bit range; eps too small" + tag)
    if flags & ERR_QUANT_RESOLUTION:
        raise QuantOverflow(
            "error bound unattainable at this precision (eps below resolution)" + tag)
    if flags & ERR_PREFIX_OVERFLOW:
        raise QuantOverflow("prefix sum overflows 63 bits" + tag)
    if flags & ERR_RESCALE_OVERFLOW:
        raise QuantOverflow("rescaled bin exceeds 63-bit range" + tag)
    if flags & ERR_OUTLIER_OVERFLOW:
        raise OutlierOverflow("outlier out of signed 32-bit range" + tag)
    if flags & ERR_OUTPUT_NONFINITE:
        raise ValueError("raw data must be finite (no NaN/Inf)" + tag)
    if flags & ERR_CAPACITY:
        raise CapacityExceeded("device output buffer too small" + tag)
    raise HoszpError(f"device error word 0x{flags:x}" + tag)
