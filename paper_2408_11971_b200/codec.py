"""Codec API -- drop-in for the reference's ``hoszp.codec`` hot path.

Same names, arguments and error behaviour as `pkg/src/hoszp/codec.py`:

==========================  ==========================  ======================
this module                 reference                   CUDA entry point
==========================  ==========================  ======================
RawArray                    codec.py:36-67              hsz_minmax (finite check)
resolve_eps                 codec.py:88-100             hsz_minmax (cached range)
quantize / dequantize       codec.py:118-160            hsz_quantize / hsz_dequantize
compress                    codec.py:495-498            hsz_compress
decompress                  codec.py:501-514            hsz_decode
decode_to_quant             codec.py:517-520            hsz_decode (bins)
encode_from_quant           codec.py:523-525            hsz_encode_bins
==========================  ==========================  ======================

Host objects in -> host objects out (each call uploads, runs the kernels,
synchronizes, checks the device error word and downloads), so code written
against the reference keeps working unchanged.  Device objects in (a
``RawArray`` built from a CUDA tensor, a :class:`DeviceStream`) -> device
objects out, asynchronously, which is how a B200 pipeline chains operations
without host round trips.  ``threads`` is accepted and ignored (results never
depended on it, codec.py:496-497).
"""

from __future__ import annotations

import numpy as np

from . import _native as N
from .device import (
    DTYPE_CODE,
    DeviceStream,
    context,
    download,
    ptr,
    require_cuda,
    run_encoder,
    torch,
)
from .errors import GeometryMismatch, raise_for_flags
from .model import DTYPES, CompressedStream, QuantArray, QuantParams

_TORCH_DTYPE = {"f32": "float32", "f64": "float64"}


def _is_cuda_tensor(x) -> bool:
    return type(x).__module__.startswith("torch") and bool(getattr(x, "is_cuda", False))


class RawArray:
    """Flat row-major array of finite reals plus its geometry
    (reference: codec.py:36-67).

    ``values`` may be a numpy array (host origin: results of operations on it
    come back as host objects) or a CUDA tensor (device origin).  The finite
    check of the reference runs on the GPU (hsz_minmax), which also caches the
    value range for :func:`resolve_eps`.
    """

    __slots__ = ("dims", "dtype", "_host", "_dev", "_range")

    def __init__(self, values, dims, dtype: str = "f32", *, _validated=False, _range=None):
        self.dims = tuple(int(d) for d in dims)
        if dtype not in DTYPES:
            raise ValueError(f"dtype must be one of {sorted(DTYPES)}, got {dtype!r}")
        self.dtype = dtype
        n = 1
        for d in self.dims:
            n *= d
        if _is_cuda_tensor(values):
            t = torch()
            dev = values.reshape(-1)
            want = getattr(t, _TORCH_DTYPE[dtype])
            if dev.dtype != want:
                dev = dev.to(want)
            self._dev = dev.contiguous()
            self._host = None
            count = self._dev.numel()
        else:
            self._host = np.ascontiguousarray(values, dtype=DTYPES[dtype][1]).ravel()
            self._dev = None
            count = self._host.shape[0]
        if count != n:
            raise ValueError(f"got {count} values for dims {self.dims}")
        self._range = _range
        if not _validated:
            self._validate()

    # -- storage -------------------------------------------------------------
    @property
    def on_device(self) -> bool:
        return self._host is None

    @property
    def values(self):
        """numpy array for host-origin arrays, CUDA tensor for device-origin."""
        return self._host if self._host is not None else self._dev

    def numpy(self) -> np.ndarray:
        if self._host is None:
            return download([self._dev])[0]
        return self._host

    def device_values(self, ctx=None):
        if self._dev is None:
            t = require_cuda()
            ctx = ctx or context()
            src = t.from_numpy(self._host)
            self._dev = t.empty(src.shape, dtype=src.dtype, device=ctx.device)
            self._dev.copy_(src, non_blocking=False)
        return self._dev

    @property
    def nbytes(self) -> int:
        return int(np.prod(self.dims, dtype=object)) * DTYPES[self.dtype][2]

    def _validate(self):
        ctx = context()
        x = self.device_values(ctx)
        lib = ctx.lib
        wsp, wsb = ctx.workspace(1, 1)
        n = x.numel()
        seq = ctx.next_seq()
        N.check(lib.hsz_minmax_mb(x.data_ptr(), DTYPE_CODE[self.dtype], n, ctx.result_ptr,
                                  ctx.err_ptr, wsp, wsb, ctx.mailbox_ptr, seq, ctx.handle),
                "hsz_minmax")
        mm = ctx.mailbox_result(seq, 2, "RawArray").view(np.float64)
        lo, hi = float(mm[0]), float(mm[1])
        self._range = (lo, hi)

    def value_range(self):
        if self._range is None:
            self._validate()
        return self._range

    def __eq__(self, other):
        if not isinstance(other, RawArray):
            return NotImplemented
        return (self.dims == other.dims and self.dtype == other.dtype
                and np.array_equal(self.numpy(), other.numpy()))

    __hash__ = None

    def __repr__(self):
        where = "device" if self.on_device else "host"
        return f"RawArray({where}, dims={self.dims}, dtype={self.dtype})"


def read_raw(path, dims, dtype: str = "f32") -> RawArray:
    """Headerless little-endian file -> RawArray (codec.py:70-80)."""
    values = np.fromfile(path, dtype="<f4" if dtype == "f32" else "<f8")
    dims = tuple(int(d) for d in dims)
    n = int(np.prod(np.asarray(dims, dtype=np.int64)))
    if values.size != n:
        raise GeometryMismatch(f"file holds {values.size} {dtype} values but dims {dims} imply {n}")
    return RawArray(values, dims, dtype)


def write_raw(raw: RawArray, path) -> None:
    """codec.py:83-85."""
    raw.numpy().astype("<f4" if raw.dtype == "f32" else "<f8").tofile(path)


def resolve_eps(raw: RawArray, eps: float, mode: str = "abs") -> float:
    """codec.py:88-100: ``rel`` scales eps by (max - min) of the data; the range
    comes from the GPU value-range pass (exact: f32 widens exactly to f64)."""
    if mode == "abs":
        return float(eps)
    if mode == "rel":
        lo, hi = raw.value_range()
        return float(eps) * (hi - lo)
    raise ValueError(f"eps mode must be 'abs' or 'rel', got {mode!r}")


def _check_geometry(raw: RawArray, params: QuantParams):
    if raw.dims != params.dims or raw.dtype != params.dtype:
        raise ValueError(f"raw geometry {raw.dims}/{raw.dtype} does not match params "
                         f"{params.dims}/{params.dtype}")


def _as_device_stream(stream) -> DeviceStream:
    if isinstance(stream, DeviceStream):
        return stream
    if isinstance(stream, CompressedStream):
        return DeviceStream.from_host(stream)
    raise TypeError(f"expected CompressedStream or DeviceStream, got {type(stream).__name__}")


# ---------------------------------------------------------------------------
# quantization (codec.py:118-160)

def quantize(raw: RawArray, params: QuantParams) -> QuantArray:
    _check_geometry(raw, params)
    ctx = context()
    x = raw.device_values(ctx)
    t = torch()
    bins = ctx.empty(params.element_count, t.int64)
    N.check(ctx.lib.hsz_quantize(ptr(x), DTYPE_CODE[params.dtype], params.element_count,
                                 params.eps, ptr(bins), ctx.err_ptr, ctx.handle), "hsz_quantize")
    if raw.on_device:
        return QuantArray(bins, params)
    ctx.check("quantize")
    return QuantArray(download([bins], ctx)[0], params)


def dequantize(q: QuantArray) -> RawArray:
    p = q.params
    ctx = context()
    t = torch()
    bins = q.bins if q.on_device else t.from_numpy(q.bins).to(ctx.device)
    kind = N.HSZ_OUT_F32 if p.dtype == "f32" else N.HSZ_OUT_F64
    out = ctx.empty(p.element_count, t.float32 if p.dtype == "f32" else t.float64)
    N.check(ctx.lib.hsz_dequantize(ptr(bins), p.element_count, p.eps, kind, ptr(out),
                                   ctx.err_ptr, ctx.handle), "hsz_dequantize")
    if q.on_device:
        return RawArray(out, p.dims, p.dtype, _validated=True)
    ctx.check("dequantize")
    return RawArray(download([out], ctx)[0], p.dims, p.dtype, _validated=True)


# ---------------------------------------------------------------------------
# compress / decompress

def compress_device(x, params: QuantParams, ctx=None) -> DeviceStream:
    """Compress a contiguous CUDA tensor (float32/float64 per params.dtype)."""
    ctx = ctx or context()
    lib = ctx.lib
    n, k = params.element_count, params.block_len
    wsp, wsb = ctx.workspace(n, k)
    xp = ptr(x)
    code = DTYPE_CODE[params.dtype]

    def launch(w, o, s, scap, p, pcap, toff):
        N.check(lib.hsz_compress(xp, code, n, k, params.eps, w, o, s, scap,
                                 p, pcap, toff, ctx.err_ptr, wsp, wsb, ctx.handle),
                "hsz_compress")

    return run_encoder(ctx, params, launch)


def compress(raw: RawArray, params: QuantParams, threads: int = 1):
    """quantize -> decorrelate -> bit-pack, one fused single-pass kernel."""
    _check_geometry(raw, params)
    ctx = context()
    ds = compress_device(raw.device_values(ctx), params, ctx)
    if raw.on_device:
        return ds
    return ds.to_host()


def decode_device(ds: DeviceStream, kind: int):
    t = torch()
    ctx = ds.ctx
    p = ds.params
    dt = {N.HSZ_OUT_F32: t.float32, N.HSZ_OUT_F64: t.float64, N.HSZ_OUT_BINS: t.int64}[kind]
    out = ctx.empty(p.element_count, dt)
    w, o, s, py, toff = ds.pointers()
    N.check(ctx.lib.hsz_decode(w, o, s, py, toff, p.element_count, p.block_len, p.eps, kind,
                               ptr(out), ctx.err_ptr, ctx.handle), "hsz_decode")
    return out


def decompress(stream, threads: int = 1, out_dtype=None) -> RawArray:
    """bit-unpack -> prefix-sum -> dequantize (codec.py:501-514)."""
    ds = _as_device_stream(stream)
    p = ds.params
    grid64 = (out_dtype is np.float64 and p.dtype == "f32") or p.dtype == "f64"
    kind = N.HSZ_OUT_F64 if grid64 else N.HSZ_OUT_F32
    out = decode_device(ds, kind)
    dtype = "f64" if grid64 else "f32"
    if isinstance(stream, DeviceStream):
        return RawArray(out, p.dims, dtype, _validated=True)
    ds.ctx.check("decompress")
    return RawArray(download([out], ds.ctx)[0], p.dims, dtype, _validated=True)


def decode_to_quant(stream, threads: int = 1) -> QuantArray:
    """Partial decode to int64 bins (codec.py:517-520)."""
    ds = _as_device_stream(stream)
    bins = decode_device(ds, N.HSZ_OUT_BINS)
    if isinstance(stream, DeviceStream):
        return QuantArray(bins, ds.params)
    ds.ctx.check("decode_to_quant")
    return QuantArray(download([bins], ds.ctx)[0], ds.params)


def encode_from_quant(q: QuantArray, threads: int = 1):
    """int64 bins -> stream (codec.py:523-525)."""
    ctx = context()
    p = q.params
    n, k = p.element_count, p.block_len
    t = torch()
    bins = q.bins if q.on_device else t.from_numpy(np.ascontiguousarray(q.bins)).to(ctx.device)
    wsp, wsb = ctx.workspace(n, k)
    lib = ctx.lib

    def launch(w, o, s, scap, py, pcap, toff):
        N.check(lib.hsz_encode_bins(ptr(bins), n, k, w, o, s, scap, py, pcap,
                                    toff, ctx.err_ptr, wsp, wsb, ctx.handle),
                "hsz_encode_bins")

    ds = run_encoder(ctx, p, launch)
    if q.on_device:
        return ds
    return ds.to_host()
