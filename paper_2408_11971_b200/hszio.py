"""Device-side stream assembly and ``.hsz`` file I/O (
reference ``model.py:299-376``, ``FORMAT.md``).

* ``serialize_device(ds)``  -- the canonical ``.hsz`` bytes of a
  DeviceStream assembled in ONE device buffer (header uploaded, the four
  sections copied device-to-device at their FORMAT.md offsets);
* ``write_hsz(stream, path)`` -- streams that buffer to a file through two
  pinned chunks (D2H of chunk i+1 overlaps the write of chunk i);
* ``read_hsz(path)`` -> DeviceStream -- the file streams into HBM through
  pinned chunks; the header is validated on the host (it is 20 + 8 ndim
  bytes), the section lengths on the device (tile-offset scan of the widths
  section), with the reference's exception classes for every malformed
  input (``BadMagic``, ``VersionMismatch``, ``TruncatedStream``,
  ``GeometryMismatch``); the sections are then laid out 256-byte aligned
  (device-to-device copies) for the decoders.

The multi-GPU writer -- every rank writes its shard's sections straight into
one shared file at the C2 offsets, no gather -- is
``sharding.Collectives.write_sharded``.
"""

from __future__ import annotations

import os

import numpy as np

from . import _native as N
from .device import DeviceStream, context, geometry, new_stream_buffers, torch
from .errors import BadMagic, GeometryMismatch, TruncatedStream, VersionMismatch
from .model import _NAME_OF_CODE, HEADER, MAGIC, VERSION, QuantParams, header_bytes, serialize

CHUNK = 64 << 20


def section_layout(params: QuantParams, sign_bytes: int, payload_bytes: int):
    """FORMAT.md offsets: (header, widths, outliers, signs, payload, end)."""
    h = len(header_bytes(params))
    B = params.block_count
    return h, h, h + B, h + 5 * B, h + 5 * B + sign_bytes, h + 5 * B + sign_bytes + payload_bytes


def serialize_device(ds: DeviceStream):
    """Canonical bytes of a device stream in one device uint8 tensor."""
    t = torch()
    ds.check()
    sb, pb = ds.totals()
    p = ds.params
    _, ow, oo, os_, op, end = section_layout(p, sb, pb)
    hdr = header_bytes(p)
    with t.cuda.stream(ds.ctx.stream):
        out = t.empty(end, dtype=t.uint8, device=ds.ctx.device)
        out[:len(hdr)].copy_(t.frombuffer(bytearray(hdr), dtype=t.uint8), non_blocking=False)
        out[ow:oo].copy_(ds.widths, non_blocking=True)
        out[oo:os_].copy_(ds.outliers.view(t.uint8), non_blocking=True)
        if sb:
            out[os_:op].copy_(ds.signs[:sb], non_blocking=True)
        if pb:
            out[op:end].copy_(ds.payload[:pb], non_blocking=True)
    return out


def write_hsz(stream, path, chunk: int = CHUNK) -> int:
    """Write a stream (host or device) as a ``.hsz`` file; returns its size."""
    if not isinstance(stream, DeviceStream):
        data = serialize(stream)
        with open(path, "wb") as f:
            f.write(data)
        return len(data)
    t = torch()
    buf = serialize_device(stream)
    total = buf.numel()
    ctx = stream.ctx
    pins = [t.empty(min(chunk, total), dtype=t.uint8, pin_memory=True) for _ in range(2)]
    evs = [None, None]
    with open(path, "wb") as f, t.cuda.stream(ctx.stream):
        pos, j = 0, 0
        pending = []
        while pos < total or pending:
            if pos < total:
                nb = min(chunk, total - pos)
                if evs[j] is not None:
                    evs[j].synchronize()
                pins[j][:nb].copy_(buf[pos:pos + nb], non_blocking=True)
                ev = t.cuda.Event()
                ev.record(ctx.stream)
                evs[j] = ev
                pending.append((j, nb, ev))
                pos += nb
                j ^= 1
            if len(pending) == 2 or pos >= total:
                jj, nb, ev = pending.pop(0)
                ev.synchronize()
                f.write(memoryview(pins[jj].numpy()[:nb]))
    return total


def _parse_header(head: bytes, size: int):
    """The reference's header checks (model.py:317-352)."""
    if size < HEADER.size:
        if head[:len(MAGIC)] != MAGIC[:len(head)]:
            raise BadMagic("not a compressed stream (magic mismatch)")
        raise TruncatedStream(f"{size} bytes is shorter than the fixed header")
    magic, version, code, ndim, eps, block_len = HEADER.unpack_from(head, 0)
    if magic != MAGIC:
        raise BadMagic(f"bad magic {magic!r}")
    if version != VERSION:
        raise VersionMismatch(f"unsupported stream version {version}")
    if code not in _NAME_OF_CODE:
        raise GeometryMismatch(f"unknown dtype code {code}")
    if ndim < 1:
        raise GeometryMismatch("header declares zero dimensions")
    if not (eps > 0.0 and np.isfinite(eps)):
        raise GeometryMismatch(f"invalid error bound {eps}")
    end = HEADER.size + 8 * ndim
    if size < end:
        raise TruncatedStream("byte sequence ends inside the dims table")
    dims = tuple(int(v) for v in np.frombuffer(head, dtype="<u8", count=ndim, offset=HEADER.size))
    if min(dims) < 1:
        raise GeometryMismatch(f"non-positive dim in {dims}")
    if block_len < 1:
        raise GeometryMismatch(f"invalid block_len {block_len}")
    return QuantParams(eps=eps, dims=dims, block_len=block_len, dtype=_NAME_OF_CODE[code]), end


def read_hsz(path, chunk: int = CHUNK) -> DeviceStream:
    """Load a ``.hsz`` file into HBM as a DeviceStream (validated like the
    reference's deserialize)."""
    t = torch()
    ctx = context()
    size = os.path.getsize(path)
    with open(path, "rb") as f:
        head = f.read(min(size, HEADER.size + 8 * 65535))
        params, pos = _parse_header(head, size)
        n, k = params.element_count, params.block_len
        B = params.block_count
        if size < pos + B:
            raise TruncatedStream("byte sequence ends inside the widths section")
        if size < pos + 5 * B:
            raise TruncatedStream("byte sequence ends inside the outliers section")
        # the whole file streams into one device staging buffer
        stage = t.empty(size + N.HSZ_SECTION_SLACK, dtype=t.uint8, device=ctx.device)
        pins = [t.empty(min(chunk, size), dtype=t.uint8, pin_memory=True) for _ in range(2)]
        evs = [None, None]
        f.seek(0)
        off, j = 0, 0
        with t.cuda.stream(ctx.stream):
            while off < size:
                nb = min(chunk, size - off)
                if evs[j] is not None:
                    evs[j].synchronize()
                f.readinto(memoryview(pins[j].numpy())[:nb])
                stage[off:off + nb].copy_(pins[j][:nb], non_blocking=True)
                ev = t.cuda.Event()
                ev.record(ctx.stream)
                evs[j] = ev
                off += nb
                j ^= 1
    with t.cuda.stream(ctx.stream):
        widths_st = stage[pos:pos + B]
        if B and int(widths_st.max().item()) > 64:
            raise GeometryMismatch("a width exceeds 64 bits")
        # section lengths from the widths (tile-offset scan on the device)
        T = geometry(n, k)[0]
        wt = t.empty(B + 16, dtype=t.uint8, device=ctx.device)
        wt[:B].copy_(widths_st, non_blocking=True)
        tt_dev = t.empty(2 * (T + 1), dtype=t.int64, device=ctx.device)
        wsp, wsb = ctx.workspace(n, k)
        N.check(ctx.lib.hsz_tile_offsets(wt.data_ptr(), n, k, tt_dev.data_ptr(), ctx.err_ptr, wsp,
                                         wsb, ctx.handle), "hsz_tile_offsets")
        (tt,) = ctx.fetch_checked([tt_dev[2 * T:2 * T + 2]], "read_hsz")
        n_sign, n_pay = int(tt.view(np.uint64)[0]), int(tt.view(np.uint64)[1])
        o_sg = pos + 5 * B
        if size < o_sg + n_sign:
            raise TruncatedStream("byte sequence ends inside the sign-plane section")
        if size < o_sg + n_sign + n_pay:
            raise TruncatedStream("byte sequence ends inside the payload section")
        if o_sg + n_sign + n_pay != size:
            raise GeometryMismatch(f"{size - (o_sg + n_sign + n_pay)} trailing bytes beyond the "
                                   "declared sections")
        # the sections laid out 256-byte aligned for the decoders
        secs, (w, o, s, py, toff), scap, pcap = new_stream_buffers(ctx, params, payload_cap=n_pay)
        buf = secs[0][0]
        buf[0:B].copy_(wt[:B], non_blocking=True)
        buf[secs[1][1]:secs[1][1] + 4 * B].copy_(stage[pos + B:pos + 5 * B], non_blocking=True)
        if n_sign:
            buf[secs[2][1]:secs[2][1] + n_sign].copy_(stage[o_sg:o_sg + n_sign], non_blocking=True)
        if n_pay:
            buf[secs[3][1]:secs[3][1] + n_pay].copy_(stage[o_sg + n_sign:size], non_blocking=True)
        buf[secs[4][1]:secs[4][1] + 16 * (T + 1)].copy_(tt_dev.view(t.uint8), non_blocking=True)
    ds = DeviceStream(params, *secs, ctx, n_sign, n_pay)
    ds._ptrs = (w, o, s, py, toff)
    ds._totals = (n_sign, n_pay)
    return ds


__all__ = ["serialize_device", "write_hsz", "read_hsz", "section_layout"]
