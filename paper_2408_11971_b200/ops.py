"""Homomorphic operations -- drop-in for the reference's ``hoszp.ops`` hot path.

==================  =====================  =================================
this module         reference              CUDA entry point
==================  =====================  =================================
ScalarBin           ops.py:51-74           (host: exact Python float/int)
negate              ops.py:88-109          hsz_negate
scalar_add / _sub   ops.py:112-125         hsz_scalar_add
scalar_mul          ops.py:199-225         hsz_scalar_mul (fused decode/encode)
elementwise_add/sub ops.py:163-192         hsz_elementwise
mean                ops.py:360-363         hsz_moments + host finalize
variance / stddev   ops.py:382-397         hsz_moments(want_sq) + finalize
apply_stream_op     ops.py:520-538         dispatch
apply_reduction     ops.py:541-552         dispatch
==================  =====================  =================================

Reductions are exact: the kernel returns S = sum(bins) (int128) and
Q = sum(bins^2) (uint192) and the final float64 arithmetic is the
reference's own Python expression on Python ints, so mean / variance are
bit-identical to the reference, not merely within tolerance.

elementwise_add / elementwise_sub (ops.py:163-192)
run as one fused pass for block_len 32; hadamard, covariance, ssim_global
and block_means (§8(f) row 3) decode their operands to int64 bins and
reduce / rescale them exactly (hsz_bivar.cuh).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .codec import _as_device_stream
from .device import DeviceStream, ptr, run_encoder, torch
from .errors import ParamsMismatch, QuantOverflow
from .model import CompressedStream

_I64_MAX = 2 ** 63 - 1

#: stream-returning operations: name -> (operand streams, takes a scalar)  (ops.py:37-45)
STREAM_OPS = {
    "neg": (1, False),
    "sadd": (1, True),
    "ssub": (1, True),
    "smul": (1, True),
    "eadd": (2, False),
    "esub": (2, False),
    "hadamard": (2, False),
}

#: scalar-returning reductions: name -> operand streams  (ops.py:48)
REDUCTIONS = {"mean": 1, "variance": 1, "stddev": 1, "covariance": 2, "ssim": 2}

#: the subset implemented by this B200 hot path (all of them)
HOT_STREAM_OPS = ("neg", "sadd", "ssub", "smul", "eadd", "esub", "hadamard")
HOT_REDUCTIONS = ("mean", "variance", "stddev", "covariance", "ssim")


@dataclass(frozen=True)
class ScalarBin:
    """A scalar on a stream's bin grid: ``trunc(s / 2eps)`` toward zero
    (reference: ops.py:51-74)."""

    value: float
    eps: float
    bin: int

    @classmethod
    def of(cls, value: float, eps: float) -> "ScalarBin":
        q = float(value) / (2.0 * eps)
        if not math.isfinite(q) or abs(q) >= 2.0 ** 63:
            raise QuantOverflow(f"scalar {value} overflows the bin grid at eps={eps}")
        return cls(float(value), float(eps), math.trunc(q))

    @property
    def quantized_value(self) -> float:
        return 2.0 * self.eps * self.bin


def _finish(stream, ds: DeviceStream, what: str):
    if isinstance(stream, DeviceStream):
        return ds
    return ds.to_host()


# ---------------------------------------------------------------------------
# fully-compressed-space operations

def negate(c):
    """Flip every stored sign bit, negate every outlier; widths, payload and
    the tile-offset cache are shared with the input (ops.py:102-109)."""
    ds = _as_device_stream(c)
    ctx = ds.ctx
    t = torch()
    p = ds.params
    B = p.block_count
    ns = ds.sign_cap + N.HSZ_SECTION_SLACK
    o_s = (4 * B + 255) & ~255
    buf = ctx.empty(o_s + ns, t.uint8)              # one allocation: outliers | signs
    base = buf.data_ptr()
    w, o, sg, py, toff = ds.pointers()
    N.check(ctx.lib.hsz_negate(w, o, base, sg, base + o_s, toff, p.element_count, p.block_len,
                               ctx.err_ptr, ctx.handle), "hsz_negate")
    out = DeviceStream(p, ds.section(0), (buf, 0, 4 * B, t.int32), (buf, o_s, ns, None),
                       ds.section(3), ds.section(4), ctx, ds.sign_cap, ds.payload_cap)
    out._ptrs = (w, base, base + o_s, py, toff)
    out._totals = ds._totals
    return _finish(c, out, "negate")


def _shift_outliers(c, rs: int, what: str):
    ds = _as_device_stream(c)
    ctx = ds.ctx
    t = torch()
    B = ds.params.block_count
    outl = ctx.empty(B, t.int32)
    w, o, sg, py, toff = ds.pointers()
    po = outl.data_ptr()
    N.check(ctx.lib.hsz_scalar_add(o, po, B, rs, ctx.err_ptr, ctx.handle), "hsz_scalar_add")
    out = DeviceStream(ds.params, ds.section(0), outl, ds.section(2), ds.section(3), ds.section(4),
                       ctx, ds.sign_cap, ds.payload_cap)
    out._ptrs = (w, po, sg, py, toff)
    out._totals = ds._totals
    return _finish(c, out, what)


def scalar_add(c, s: float):
    """Shift every outlier by the scalar's bin (ops.py:112-118)."""
    eps = c.params.eps
    return _shift_outliers(c, ScalarBin.of(s, eps).bin, "scalar_add")


def scalar_sub(c, s: float):
    """ops.py:121-125."""
    eps = c.params.eps
    return _shift_outliers(c, -ScalarBin.of(s, eps).bin, "scalar_sub")


# ---------------------------------------------------------------------------
# residual-space operations on two streams

def _check_params(a, b):
    """ops.py:77-81."""
    if a.params != b.params:
        raise ParamsMismatch(f"operand params differ: {a.params} vs {b.params}")


def _elementwise(a, b, sub: bool, what: str):
    """ops.py:163-182: outliers combine (int32 guard on the result), signed
    residuals combine element by element, the result is re-encoded."""
    _check_params(a, b)
    da = _as_device_stream(a)
    db = _as_device_stream(b)
    ctx = da.ctx
    lib = ctx.lib
    p = da.params
    n, k = p.element_count, p.block_len
    wsp, wsb = ctx.workspace(n, k)
    scratch_bytes = int(lib.hsz_elementwise_scratch_size(n, k))
    scratch = ctx.empty(scratch_bytes, torch().uint8) if scratch_bytes else None
    sp = ptr(scratch) if scratch is not None else None
    wa, oa, sa, pa, ta = da.pointers()
    wb, ob, sb, pb, tb = db.pointers()

    def launch(ow, oo, os_, scap, op, pcap, otoff):
        N.check(lib.hsz_elementwise(wa, oa, sa, pa, ta, wb, ob, sb, pb, tb, n, k, 1 if sub else 0,
                                    ow, oo, os_, scap, op, pcap, otoff, sp,
                                    ctx.err_ptr, wsp, wsb, ctx.handle), "hsz_elementwise")

    out = run_encoder(ctx, p, launch)
    return _finish(a, out, what)


def elementwise_add(a, b, threads: int = 1):
    """Per block: outliers add, signed residuals add; the result decompresses
    to the exact sum of the operands' reconstructions (ops.py:185-188)."""
    return _elementwise(a, b, False, "elementwise_add")


def elementwise_sub(a, b, threads: int = 1):
    """ops.py:191-192."""
    return _elementwise(a, b, True, "elementwise_sub")


# ---------------------------------------------------------------------------
# quantized-space operations

def scalar_mul(c, s: float, threads: int = 1):
    """bins * rs, re-centred with nearest-ties-away rounding, re-encoded --
    one fused single-pass kernel for block_len 32 (ops.py:211-225)."""
    p = c.params
    rs = ScalarBin.of(s, p.eps).bin
    ds = _as_device_stream(c)
    ctx = ds.ctx
    lib = ctx.lib
    n, k = p.element_count, p.block_len
    wsp, wsb = ctx.workspace(n, k)
    scratch_bytes = int(lib.hsz_scalar_mul_scratch_size(n, k))
    scratch = ctx.empty(scratch_bytes, torch().uint8) if scratch_bytes else None
    sp = ptr(scratch) if scratch is not None else None
    w, o, sg, py, toff = ds.pointers()

    def launch(ow, oo, os_, scap, op, pcap, otoff):
        N.check(lib.hsz_scalar_mul(w, o, sg, py, toff, n, k, p.eps, rs, ow, oo,
                                   os_, scap, op, pcap, otoff, sp, ctx.err_ptr,
                                   wsp, wsb, ctx.handle), "hsz_scalar_mul")

    out = run_encoder(ctx, p, launch)
    return _finish(c, out, "scalar_mul")


# ---------------------------------------------------------------------------
# bivariate quantized-domain operations

def _bivar_scratch(ctx, n, k):
    return ctx.empty(int(ctx.lib.hsz_bivariate_scratch_size(n, k)), torch().uint8)


def hadamard(a, b, threads: int = 1):
    """Element-wise product via the quantized domain: the scalar-multiply
    rescale rule with b's bins as the scalars (ops.py:226-240)."""
    _check_params(a, b)
    da, db = _as_device_stream(a), _as_device_stream(b)
    ctx = da.ctx
    p = da.params
    n, k = p.element_count, p.block_len
    wsp, wsb = ctx.workspace(n, k)
    scratch = _bivar_scratch(ctx, n, k)
    sp = ptr(scratch)
    wa, oa, sa, pa, ta = da.pointers()
    wb, ob, sb, pb, tb = db.pointers()

    def launch(ow, oo, os_, scap, op, pcap, otoff):
        N.check(ctx.lib.hsz_hadamard(wa, oa, sa, pa, ta, wb, ob, sb, pb, tb, n, k, p.eps, ow, oo,
                                     os_, scap, op, pcap, otoff, sp, ctx.err_ptr, wsp, wsb,
                                     ctx.handle), "hsz_hadamard")

    out = run_encoder(ctx, p, launch)
    return _finish(a, out, "hadamard")


def _bank(c, j0, nchunks) -> int:
    return sum(c[j0 + j] << (32 * j) for j in range(nchunks))


def pair_stats(a, b):
    """Exact integer (S_a, Q_a, min_a, max_a, S_b, Q_b, min_b, max_b, S_ab)
    over the bins of two streams -- the sums behind covariance and
    ssim_global (ops.py:313-357, 361-450)."""
    _check_params(a, b)
    da, db = _as_device_stream(a), _as_device_stream(b)
    ctx = da.ctx
    p = da.params
    n, k = p.element_count, p.block_len
    scratch = _bivar_scratch(ctx, n, k)
    out = ctx.empty(52, torch().int64)
    N.check(ctx.lib.hsz_pair_stats(*da.pointers(), *db.pointers(), n, k, ptr(out), ptr(scratch),
                                   ctx.err_ptr, ctx.handle), "hsz_pair_stats")
    (w,) = ctx.fetch_checked([out], "pair_stats")
    u = [int(x) for x in np.asarray(w).view(np.uint64)]
    c = [u[2 * j] + (u[2 * j + 1] << 32) for j in range(24)]
    mm = [int(x) for x in np.asarray(w)[48:52]]
    sa = _bank(c, 0, 2) - _bank(c, 2, 2)
    sb = _bank(c, 4, 2) - _bank(c, 6, 2)
    return (sa, _bank(c, 8, 4), mm[0], mm[1], sb, _bank(c, 12, 4), mm[2], mm[3],
            _bank(c, 16, 4) - _bank(c, 20, 4))


def covariance(a, b, *, shortcut: bool = True, threads: int = 1) -> float:
    """Population covariance via exact integer sums (ops.py:453-462)."""
    _check_params(a, b)
    n = a.params.element_count
    sa, _, _, _, sb, _, _, _, sab = pair_stats(a, b)
    return (2.0 * a.params.eps) ** 2 * float(n * sab - sa * sb) / (n * n)


def ssim_global(a, b, *, threads: int = 1) -> float:
    """Single global SSIM from the exact quantized-domain sums, with the
    reference's float expressions (ops.py:465-487)."""
    _check_params(a, b)
    n = a.params.element_count
    eps2 = 2.0 * a.params.eps
    sa, sqa, lo_a, hi_a, sb, sqb, lo_b, hi_b, sab = pair_stats(a, b)
    mu_a = eps2 * sa / n
    mu_b = eps2 * sb / n
    var_a = eps2**2 * float(n * sqa - sa * sa) / (n * n)
    var_b = eps2**2 * float(n * sqb - sb * sb) / (n * n)
    cov = eps2**2 * float(n * sab - sa * sb) / (n * n)
    value_range = eps2 * max(hi_a - lo_a, hi_b - lo_b)
    c1 = (0.01 * value_range) ** 2
    c2 = (0.03 * value_range) ** 2
    num = (2.0 * mu_a * mu_b + c1) * (2.0 * cov + c2)
    den = (mu_a * mu_a + mu_b * mu_b + c1) * (var_a + var_b + c2)
    if den == 0.0:
        raise ValueError("SSIM is undefined: degenerate zero-range operands")
    return num / den


def block_means(c, threads: int = 1):
    """Per-block means 2 eps * sum(block bins) / block length
    (ops.py:366-379); numpy float64[B] for a host stream, a device tensor for
    a DeviceStream."""
    ds = _as_device_stream(c)
    ctx = ds.ctx
    p = ds.params
    n, k = p.element_count, p.block_len
    out = ctx.empty(p.block_count, torch().float64)
    scratch = ctx.empty(8 * n, torch().uint8)
    N.check(ctx.lib.hsz_block_means(*ds.pointers(), n, k, p.eps, ptr(out), ptr(scratch),
                                    ctx.err_ptr, ctx.handle), "hsz_block_means")
    if isinstance(c, DeviceStream):
        return out
    (v,) = ctx.fetch_checked([out], "block_means")
    return np.asarray(v, dtype=np.float64)


# ---------------------------------------------------------------------------
# reductions

def moments_device(ds: DeviceStream, want_sq: bool):
    """Launch the exact-moment kernel; returns the device u64[5] result."""
    ctx = ds.ctx
    p = ds.params
    n, k = p.element_count, p.block_len
    wsp, wsb = ctx.workspace(n, k)
    out = ctx.empty(5, torch().int64)
    w, o, sg, py, toff = ds.pointers()
    N.check(ctx.lib.hsz_moments(w, o, sg, py, toff, n, k, 1 if want_sq else 0, ptr(out),
                                ctx.err_ptr, wsp, wsb, ctx.handle), "hsz_moments")
    return out


def unpack_moments(limbs) -> tuple:
    """u64[5] -> (S: signed 128-bit, Q: unsigned 192-bit) as Python ints."""
    v = np.asarray(limbs).view(np.uint64).tolist()   # (Python ints; 4 us less than a per-element int())
    S = v[0] | (v[1] << 64)
    if S >= 1 << 127:
        S -= 1 << 128
    Q = v[2] | (v[3] << 64) | (v[4] << 128)
    return S, Q


def exact_moments(c, want_sq: bool = True):
    """Exact (sum(bins), sum(bins^2)) of a stream (ops.py:313-357)."""
    ds = _as_device_stream(c)
    ctx = ds.ctx
    p = ds.params
    n, k = p.element_count, p.block_len
    wsp, wsb = ctx.workspace(n, k)
    w, o, sg, py, toff = ds.pointers()
    seq = ctx.next_seq()
    N.check(ctx.lib.hsz_moments_mb(w, o, sg, py, toff, n, k, 1 if want_sq else 0, ctx.result_ptr,
                                   ctx.err_ptr, wsp, wsb, ctx.mailbox_ptr, seq, ctx.handle),
            "hsz_moments")
    return unpack_moments(ctx.mailbox_result(seq, 5, "moments"))


def mean_from(S: int, n: int, eps: float) -> float:
    """ops.py:363, evaluated with the reference's Python operators."""
    return (2.0 * eps * S) / n


def variance_from(S: int, Q: int, n: int, eps: float) -> float:
    """ops.py:386 and 393."""
    spread = float(n * Q - S * S) / (n * n)
    return (2.0 * eps) ** 2 * spread


def mean(c, *, shortcut: bool = True, threads: int = 1) -> float:
    S, _ = exact_moments(c, want_sq=False)
    return mean_from(S, c.params.element_count, c.params.eps)


def variance(c, *, shortcut: bool = True, threads: int = 1) -> float:
    S, Q = exact_moments(c, want_sq=True)
    return variance_from(S, Q, c.params.element_count, c.params.eps)


def stddev(c, *, shortcut: bool = True, threads: int = 1) -> float:
    return math.sqrt(variance(c, shortcut=shortcut, threads=threads))


# ---------------------------------------------------------------------------
# dispatch (ops.py:520-552)

def apply_stream_op(name: str, streams, scalar=None, threads: int = 1):
    arity, needs_scalar = STREAM_OPS[name]
    if len(streams) != arity:
        raise ValueError(f"{name} takes {arity} stream operand(s), got {len(streams)}")
    if needs_scalar and scalar is None:
        raise ValueError(f"{name} needs a scalar operand")
    if name == "neg":
        return negate(streams[0])
    if name == "sadd":
        return scalar_add(streams[0], scalar)
    if name == "ssub":
        return scalar_sub(streams[0], scalar)
    if name == "smul":
        return scalar_mul(streams[0], scalar, threads)
    if name == "eadd":
        return elementwise_add(streams[0], streams[1], threads)
    if name == "esub":
        return elementwise_sub(streams[0], streams[1], threads)
    if name == "hadamard":
        return hadamard(streams[0], streams[1], threads)
    raise NotImplementedError(f"stream op {name!r} is outside the B200 hot path "
                              f"(implemented: {', '.join(HOT_STREAM_OPS)})")


def apply_reduction(name: str, streams, threads: int = 1) -> float:
    if len(streams) != REDUCTIONS[name]:
        raise ValueError(f"{name} takes {REDUCTIONS[name]} stream operand(s)")
    if name == "mean":
        return mean(streams[0], threads=threads)
    if name == "variance":
        return variance(streams[0], threads=threads)
    if name == "stddev":
        return stddev(streams[0], threads=threads)
    if name == "covariance":
        return covariance(streams[0], streams[1], threads=threads)
    if name == "ssim":
        return ssim_global(streams[0], streams[1], threads=threads)
    raise NotImplementedError(f"reduction {name!r} is outside the B200 hot path "
                              f"(implemented: {', '.join(HOT_REDUCTIONS)})")


__all__ = [
    "STREAM_OPS", "REDUCTIONS", "ScalarBin", "negate", "scalar_add", "scalar_sub", "scalar_mul",
    "elementwise_add", "elementwise_sub", "hadamard", "covariance", "ssim_global", "block_means",
    "pair_stats",
    "mean", "variance", "stddev", "exact_moments", "apply_stream_op", "apply_reduction",
    "CompressedStream",
]
