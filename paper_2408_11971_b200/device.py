"""Device-resident stream and the per-CUDA-stream execution context.

:class:`DeviceStream` is the HBM twin of :class:`model.CompressedStream`:
the four FORMAT.md sections live in device buffers (torch tensors used as
plain allocations) plus a cached tile-offset table (the exclusive byte
offsets of every HSZ_TILE_BLOCKS-block tile, written for free by the
encoders' look-back).  Operations on DeviceStreams are asynchronous on the
current CUDA stream; failures are accumulated in a sticky device error word
that is checked (and raised as the reference's exception class) whenever a
result is materialised on the host (``to_host()``, a reduction's float,
``check()``).

Memory layout in HBM per stream (N elements, B blocks, T tiles):
  widths u8[B] | outliers i32[B] | signs u8[cap_s + 16] | payload u8[cap_p + 16]
  | tile offsets u64[2(T+1)]
negate / scalar_add share the untouched sections (widths, payload, tile
offsets; and signs for scalar_add) with their input, exactly like the
reference shares the numpy arrays / bytes objects (ops.py:106-118).
"""

from __future__ import annotations

import functools
import threading

import numpy as np

from . import _native as N
from .errors import ERR_LOOKBACK_TIMEOUT, CapacityExceeded, raise_for_flags
from .model import CompressedStream, QuantParams

_torch = None


def torch():
    global _torch
    if _torch is None:
        import torch as t

        _torch = t
    return _torch


_CUDA_OK = False


def require_cuda():
    global _CUDA_OK
    t = torch()
    if not _CUDA_OK:
        if not t.cuda.is_available():
            raise RuntimeError("paper_2408_11971_b200 needs a CUDA device (B200, sm_100a); "
                               "there is no CPU fallback")
        _CUDA_OK = True
    return t


@functools.lru_cache(maxsize=256)
def geometry(n: int, k: int):
    """(tiles, sign bound, payload bound, workspace bytes) for n elements of
    block length k (C-ABI queries, cached)."""
    lib = N.load()
    return (int(lib.hsz_tile_count(n, k)), int(lib.hsz_sign_bound(n, k)),
            int(lib.hsz_payload_bound(n, k)), int(lib.hsz_workspace_size(n, k)))


def ptr(t) -> int:
    return int(t.data_ptr())


DTYPE_CODE = {"f32": N.HSZ_F32, "f64": N.HSZ_F64}

# payload capacity policy: the exact worst case (8 bytes/element) up to 2 GiB
# (fields up to 2^28 values, every single-GPU config), else 2 bytes/element
# (16-bit mean width; the 2048^3 config-5 field needs ~1.1) with an
# exact-size retry on overflow -- a whole-field config-5 chain on one GPU
# then fits 180 GB of HBM, and so do shards of it sharing one GPU
_PAYLOAD_BOUND_LIMIT = 2 << 30
_PAYLOAD_BIG_BYTES_PER_ELEM = 2
_WS_REINIT_USES = 1 << 22


class Context:
    """Workspace, error word and scratch for one (device, CUDA stream)."""

    def __init__(self, device_index: int, stream):
        t = require_cuda()
        self.lib = N.load()
        self.device = t.device("cuda", device_index)
        self.stream = stream
        self.handle = int(stream.cuda_stream)
        self.ws = None
        self.ws_bytes = 0
        self.ws_uses = 0
        with t.cuda.device(self.device):
            # one small device record: [0, 16) the sticky error word(s),
            # [16, 64) the result slot of value-range / moment reductions, so a
            # reduction comes back with its error word in ONE copy
            self.small = t.zeros(8, dtype=t.int64, device=self.device)
        self.err = self.small[:2].view(t.int32)
        self.err_ptr = self.small.data_ptr()
        self.result_ptr = self.err_ptr + 16
        self._scratch = t.empty(1 << 12, dtype=t.uint8, pin_memory=True)   # small fetches
        self._scratch_np = self._scratch.numpy()
        self._scratch_ptr = self._scratch.data_ptr()
        # host-mapped mailbox (pinned, device-visible through UVA) the
        # reduction kernels post their result + error word into
        self._mailbox = t.zeros(8, dtype=t.int64, pin_memory=True)
        self.mailbox_ptr = self._mailbox.data_ptr()
        self._mailbox_np = self._mailbox.numpy().view(np.uint64)
        self.mailbox_seq = 0
        # pinned ring for asynchronous section-total copies (prefetch_totals):
        # slot = [sign total, payload total, error word, pad]
        self._tot = t.zeros(4 * _TOT_SLOTS, dtype=t.int64, pin_memory=True)
        self._tot_np = self._tot.numpy()
        self._tot_ptr = self._tot.data_ptr()
        self._tot_ev = [None] * _TOT_SLOTS
        self._tot_next = 0
        self._side = None

    def workspace(self, n: int, k: int):
        need = geometry(n, k)[3]
        self.ws_uses += 1
        if self.ws_uses >= _WS_REINIT_USES and self.ws is not None:
            # look-back words carry a 24-bit launch-epoch tag: re-zero the
            # workspace well before the tag could repeat (hsz_b200.h)
            N.check(self.lib.hsz_workspace_init(ptr(self.ws), self.ws_bytes, self.handle),
                    "workspace init")
            self.ws_uses = 0
        if need > self.ws_bytes:
            t = torch()
            need = max(need, 2 * self.ws_bytes)
            self.ws = t.empty(need, dtype=t.uint8, device=self.device)
            N.check(self.lib.hsz_workspace_init(ptr(self.ws), need, self.handle), "workspace init")
            self.ws_bytes = need
        return ptr(self.ws), self.ws_bytes

    def synchronize(self):
        """Wait for the stream, bounded (hsz_stream_sync: a hung kernel raises
        DeviceTimeout instead of blocking forever)."""
        N.check(self.lib.hsz_stream_sync(self.handle), "stream sync")

    def raise_flags(self, flags: int, what: str = "") -> None:
        """raise_for_flags, after re-initialising the workspace when an
        encoder's look-back watchdog fired (its tickets / epoch may be left
        inconsistent; the next launch must start from a clean slate)."""
        if flags & ERR_LOOKBACK_TIMEOUT and self.ws is not None:
            self.synchronize()
            N.check(self.lib.hsz_workspace_init(ptr(self.ws), self.ws_bytes, self.handle),
                    "workspace init")
            self.synchronize()
            self.ws_uses = 0
        raise_for_flags(flags, what)

    def read_flags(self) -> int:
        """Synchronize, read and clear the sticky error word."""
        self.synchronize()
        v = int(self.err[0].item())
        if v:
            self.err.zero_()
            self.synchronize()
        return v

    def check(self, what: str = "") -> None:
        self.raise_flags(self.read_flags(), what)

    def next_seq(self) -> int:
        self.mailbox_seq += 1
        return self.mailbox_seq

    def mailbox_result(self, seq: int, nwords: int, what: str = ""):
        """Wait for the reduction that posts `seq` into the mailbox; returns
        its `nwords` result words (numpy uint64 copy).  Raises the reference's
        exception for a set error word; falls back to a copy of the result
        slot if the stream drained without a post."""
        rc = self.lib.hsz_mailbox_wait(self.mailbox_ptr, seq, self.handle)
        if rc != N.HSZ_OK:
            if rc == N.HSZ_EINVAL:
                return self.fetch_result(8 * nwords, what).view(np.uint64)
            N.check(rc, f"{what}: mailbox wait")      # DeviceTimeout on a hung kernel
            self.synchronize()                        # surfaces the CUDA error
            raise RuntimeError(f"{what}: stream failed while waiting for the result")
        mb = self._mailbox_np
        flags = int(mb[1 + nwords]) & 0xFFFFFFFF
        if flags:
            self.err.zero_()
            self.synchronize()
            self.raise_flags(flags, what)
        return mb[1:1 + nwords].copy()

    def fetch_result(self, nbytes: int, what: str = ""):
        """Wait for the result slot (``result_ptr``, ``nbytes`` <= 48) and the
        error word: one copy + synchronize; raise the reference's exception
        for a set error word.  Returns a numpy uint8 copy of the result."""
        N.check(self.lib.hsz_fetch(self._scratch_ptr, self.err_ptr, 16 + nbytes, self.handle),
                "fetch")
        host = self._scratch_np
        flags = int(host[:4].view(np.int32)[0])
        if flags:
            self.err.zero_()
            self.synchronize()
            self.raise_flags(flags, what)
        return host[16:16 + nbytes].copy()

    def fetch_checked(self, tensors, what: str = ""):
        """Download (small) `tensors` together with the sticky error word in
        ONE synchronize (C-ABI copies into a pinned scratch); raise the
        reference's exception for a set error word.  Returns numpy copies."""
        tensors = list(tensors) + [self.err]
        sizes = [int(x.numel()) * x.element_size() for x in tensors]
        total = sum((nb + 15) & ~15 for nb in sizes)
        if total > self._scratch.numel():
            self._scratch = torch().empty(max(total, 2 * self._scratch.numel()), dtype=torch().uint8,
                                          pin_memory=True)
        base = self._scratch.data_ptr()
        off = 0
        offs = []
        for x, nb in zip(tensors, sizes):
            if nb:
                N.check(self.lib.hsz_copy_d2h(base + off, x.data_ptr(), nb, self.handle), "d2h copy")
            offs.append(off)
            off += (nb + 15) & ~15
        N.check(self.lib.hsz_stream_sync(self.handle), "stream sync")
        host = self._scratch.numpy()
        out = []
        for x, nb, o in zip(tensors, sizes, offs):
            out.append(host[o:o + nb].copy().view(_NP_OF[x.dtype]))
        flags = int(out[-1][0])
        if flags:
            self.err.zero_()
            self.stream.synchronize()
            self.raise_flags(flags, what)
        return out[:-1]

    def empty(self, n, dtype):
        t = torch()
        return t.empty(int(n), dtype=dtype, device=self.device)

    def side_stream(self):
        """A second CUDA stream on this context's device (small copies that
        must not delay the main stream)."""
        if self._side is None:
            self._side = torch().cuda.Stream(device=self.device)
        return self._side

    def totals_slot(self):
        """Next slot of the pinned totals ring (waits only if the slot's
        previous copy is still in flight)."""
        i = self._tot_next
        self._tot_next = (i + 1) % _TOT_SLOTS
        if self._tot_ev[i] is not None:
            self._tot_ev[i].synchronize()
            self._tot_ev[i] = None
        return i


_TOT_SLOTS = 64


_CTX = {}
_CTX_LOCK = threading.Lock()


def context(device=None) -> Context:
    """Context of the current CUDA stream on ``device`` (default: current)."""
    t = require_cuda()
    if device is None:
        idx = t.cuda.current_device()
    else:
        idx = t.device(device).index
        if idx is None:
            idx = t.cuda.current_device()
    raw = _raw_stream(idx)
    key = (idx, raw)
    ctx = _CTX.get(key)
    if ctx is None:
        with _CTX_LOCK:
            ctx = _CTX.get(key)
            if ctx is None:
                ctx = Context(idx, t.cuda.current_stream(idx))
                _CTX[key] = ctx
    return ctx


def _raw_stream(idx: int) -> int:
    t = torch()
    fn = getattr(t._C, "_cuda_getCurrentRawStream", None)
    if fn is not None:
        return int(fn(idx))
    return int(t.cuda.current_stream(idx).cuda_stream)


def payload_capacity(lib, n: int, k: int) -> int:
    bound = int(lib.hsz_payload_bound(n, k))
    if bound <= _PAYLOAD_BOUND_LIMIT:
        return bound
    return max(_PAYLOAD_BIG_BYTES_PER_ELEM * n, 1 << 20)


class DeviceStream:
    """A compressed stream resident in HBM (see module docstring).

    Sections are held as (base tensor, byte offset, bytes, dtype) and
    materialised as torch views only when asked for (``widths`` ...); the
    launch path works on raw pointers (base pointer + offset), so an op costs
    one device allocation and no tensor slicing on the host."""

    __slots__ = ("params", "_sec", "_views", "ctx", "sign_cap", "payload_cap", "_totals", "_ptrs",
                 "_tot_pending")

    _NAMES = ("widths", "outliers", "signs", "payload", "toff")

    def __init__(self, params: QuantParams, widths, outliers, signs, payload, toff, ctx: Context,
                 sign_cap: int, payload_cap: int):
        self.params = params
        secs = (widths, outliers, signs, payload, toff)
        self._sec = secs
        self._views = [x if not isinstance(x, tuple) else None for x in secs]
        self.ctx = ctx
        self.sign_cap = int(sign_cap)
        self.payload_cap = int(payload_cap)
        self._totals = None
        self._ptrs = None
        self._tot_pending = None

    def section(self, i):
        """Section i as an aliasable descriptor (tensor or (base, off, bytes, dtype))."""
        return self._sec[i]

    def _view(self, i):
        v = self._views[i]
        if v is None:
            base, off, nb, dt = self._sec[i]
            v = base[off:off + nb]
            if dt is not None:
                v = v.view(dt)
            self._views[i] = v
        return v

    widths = property(lambda self: self._view(0))
    outliers = property(lambda self: self._view(1))
    signs = property(lambda self: self._view(2))
    payload = property(lambda self: self._view(3))
    toff = property(lambda self: self._view(4))

    # -- geometry ---------------------------------------------------------
    @property
    def n(self) -> int:
        return self.params.element_count

    @property
    def k(self) -> int:
        return self.params.block_len

    @property
    def ntiles(self) -> int:
        return geometry(self.n, self.k)[0]

    def pointers(self):
        if self._ptrs is None:
            self._ptrs = tuple((x[0].data_ptr() + x[1]) if isinstance(x, tuple) else x.data_ptr()
                               for x in self._sec)
        return self._ptrs

    # -- host materialisation ------------------------------------------------
    def check(self) -> "DeviceStream":
        """Synchronize and raise any pending device error."""
        self.ctx.check()
        return self

    def prefetch_totals(self) -> "DeviceStream":
        """Start copying the section totals (and the sticky error word) to
        pinned host memory, asynchronously on the stream; a later
        ``totals()`` then costs no device round trip once the stream has
        passed this point (e.g. after any later synchronising call)."""
        if self._totals is not None or self._tot_pending is not None:
            return self
        ctx = self.ctx
        t = torch()
        i = ctx.totals_slot()
        host = ctx._tot_ptr + 32 * i
        T = self.ntiles
        # the copies run on a side stream that waits for the producer, so the
        # main stream's next kernel does not queue behind two DMA latencies
        side = ctx.side_stream()
        side.wait_stream(ctx.stream)
        h = int(side.cuda_stream)
        N.check(ctx.lib.hsz_copy_d2h(host, self.pointers()[4] + 16 * T, 16, h), "d2h copy")
        N.check(ctx.lib.hsz_copy_d2h(host + 16, ctx.err_ptr, 4, h), "d2h copy")
        sec = self._sec[4]
        (sec[0] if isinstance(sec, tuple) else sec).record_stream(side)
        ev = t.cuda.Event()
        ev.record(side)
        ctx._tot_ev[i] = ev
        self._tot_pending = (i, ev)
        return self

    def totals(self):
        """(sign bytes, payload bytes) -- synchronizes (unless prefetched)."""
        if self._totals is None and self._tot_pending is not None:
            i, ev = self._tot_pending
            self._tot_pending = None
            ctx = self.ctx
            if ctx._tot_ev[i] is ev:             # else: the ring slot was reused; fetch below
                ev.synchronize()
                row = ctx._tot_np[4 * i:4 * i + 3].copy()
                ctx._tot_ev[i] = None
            else:
                row = None
        else:
            row = None
        if row is not None:
            flags = int(row[2]) & 0xFFFFFFFF
            if flags:
                ctx.err.zero_()
                ctx.stream.synchronize()
                ctx.raise_flags(flags, "totals")
            self._totals = (int(row[0]), int(row[1]))
        if self._totals is None:
            T = self.ntiles
            (tt,) = self.ctx.fetch_checked([self.toff[2 * T:2 * T + 2]])
            tt = tt.view(np.uint64)
            self._totals = (int(tt[0]), int(tt[1]))
        return self._totals

    @property
    def serialized_size(self) -> int:
        s, p = self.totals()
        from .model import HEADER
        return HEADER.size + 8 * len(self.params.dims) + 5 * self.params.block_count + s + p

    @property
    def compression_ratio(self) -> float:
        return self.params.raw_nbytes / self.serialized_size

    def to_host(self) -> CompressedStream:
        self.ctx.check()
        s, p = self.totals()
        w, o, sg, py = download([self.widths, self.outliers.view(torch().uint8), self.signs[:s],
                                 self.payload[:p]], self.ctx)
        return CompressedStream(self.params, w, o.view(np.int32), sg, py)

    @classmethod
    def from_host(cls, cs: CompressedStream, ctx: Context = None) -> "DeviceStream":
        """Upload a host stream and rebuild its tile-offset cache on device."""
        t = require_cuda()
        ctx = ctx or context()
        p = cs.params
        n, k = p.element_count, p.block_len
        lib = ctx.lib
        dev = ctx.device

        def up(arr_u8, extra=0):
            host = t.from_numpy(np.frombuffer(arr_u8, dtype=np.uint8).copy())
            out = t.empty(host.numel() + extra, dtype=t.uint8, device=dev)
            if host.numel():
                out[:host.numel()].copy_(host, non_blocking=False)
            return out

        widths = up(cs.widths.tobytes())
        outliers = up(cs.outliers.astype("<i4").tobytes()).view(t.int32)
        signs = up(cs.sign_planes, N.HSZ_SECTION_SLACK)
        payload = up(cs.payload, N.HSZ_SECTION_SLACK)
        T = int(lib.hsz_tile_count(n, k))
        toff = t.empty(2 * (T + 1), dtype=t.int64, device=dev)
        wsp, wsb = ctx.workspace(n, k)
        N.check(lib.hsz_tile_offsets(ptr(widths), n, k, ptr(toff), ctx.err_ptr, wsp, wsb,
                                     ctx.handle), "hsz_tile_offsets")
        ds = cls(p, widths, outliers, signs, payload, toff, ctx, len(cs.sign_planes),
                 len(cs.payload))
        ds._totals = (len(cs.sign_planes), len(cs.payload))
        return ds

    @classmethod
    def from_sections(cls, params: QuantParams, widths, outliers, signs, payload,
                      ctx: Context = None) -> "DeviceStream":
        """A stream from its four sections given as device uint8 tensors
        (e.g. views into a collective's receive buffer): copied into one
        256-byte aligned allocation with the decoders' slack, tile-offset
        cache rebuilt on the device.  Asynchronous; the section lengths are
        the caller's (checked against the widths by the tile-offset totals
        only when ``totals()`` is asked for)."""
        t = require_cuda()
        ctx = ctx or context()
        n, k = params.element_count, params.block_len
        B = params.block_count
        ns, npay = int(signs.numel()), int(payload.numel())
        secs, (w, o, s, py, toff), scap, pcap = new_stream_buffers(ctx, params, payload_cap=npay)
        buf = secs[0][0]
        with t.cuda.stream(ctx.stream):
            buf[0:B].copy_(widths, non_blocking=True)
            buf[secs[1][1]:secs[1][1] + 4 * B].copy_(outliers, non_blocking=True)
            if ns:
                buf[secs[2][1]:secs[2][1] + ns].copy_(signs, non_blocking=True)
            if npay:
                buf[secs[3][1]:secs[3][1] + npay].copy_(payload, non_blocking=True)
        wsp, wsb = ctx.workspace(n, k)
        N.check(ctx.lib.hsz_tile_offsets(w, n, k, toff, ctx.err_ptr, wsp, wsb, ctx.handle),
                "hsz_tile_offsets")
        ds = cls(params, *secs, ctx, scap, pcap)
        ds._ptrs = (w, o, s, py, toff)
        ds._totals = (ns, npay)
        return ds

    def __eq__(self, other):
        if isinstance(other, DeviceStream):
            other = other.to_host()
        if not isinstance(other, CompressedStream):
            return NotImplemented
        return self.to_host() == other

    __hash__ = None

    def __repr__(self):
        return f"DeviceStream({self.params}, device={self.ctx.device})"


_PINNED = {}
_NP_OF_NAMES = {"uint8": np.uint8, "int32": np.int32, "int64": np.int64, "float32": np.float32,
                "float64": np.float64}


class _NpOf(dict):
    def __missing__(self, dt):
        v = _NP_OF_NAMES[str(dt).split(".")[-1]]
        self[dt] = v
        return v


_NP_OF = _NpOf()


def download(tensors, ctx: Context = None):
    """Copy device tensors to host numpy arrays through one pinned staging
    buffer (one async copy each, one synchronize).  The arrays are copies."""
    t = torch()
    sizes = [int(x.numel()) * x.element_size() for x in tensors]
    total = sum(sizes)
    key = t.cuda.current_device() if ctx is None else ctx.device.index
    buf = _PINNED.get(key)
    if buf is None or buf.numel() < total:
        buf = t.empty(max(total, 1 << 20), dtype=t.uint8, pin_memory=True)
        _PINNED[key] = buf
    off = 0
    views = []
    for x, nb in zip(tensors, sizes):
        dst = buf[off:off + nb]
        if nb:
            dst.copy_(x.reshape(-1).view(t.uint8), non_blocking=True)
        views.append((off, nb, x.dtype))
        off += nb
    (ctx.stream if ctx is not None else t.cuda.current_stream()).synchronize()
    host = buf.numpy()
    out = []
    for (o, nb, dt), x in zip(views, tensors):
        a = host[o:o + nb].copy()
        npdt = {t.uint8: np.uint8, t.int32: np.int32, t.int64: np.int64, t.float32: np.float32,
                t.float64: np.float64}[dt]
        out.append(a.view(npdt))
    return out


def download_into(tensors, arena, ctx: Context = None):
    """Copy device tensors into a caller-owned pinned host arena (uint8 CPU
    tensor): one async copy each, one synchronize.  Returns numpy views into
    the arena (valid until the arena is reused)."""
    t = torch()
    off = 0
    views = []
    for x in tensors:
        nb = int(x.numel()) * x.element_size()
        if nb:
            arena[off:off + nb].copy_(x.reshape(-1).view(t.uint8), non_blocking=True)
        views.append((off, nb))
        off += (nb + 15) & ~15
    (ctx.stream if ctx is not None else t.cuda.current_stream()).synchronize()
    host = arena.numpy()
    return [host[o:o + nb] for o, nb in views]


def new_stream_buffers(ctx: Context, params: QuantParams, payload_cap: int = None):
    """Allocate output sections for an encoder writing `params`-shaped data:
    ONE device allocation carved into 256-byte aligned sections (returned as
    section descriptors; no views are made here)."""
    t = torch()
    n, k = params.element_count, params.block_len
    B = params.block_count
    T, scap, pbound, _ = geometry(n, k)
    pcap = payload_capacity(ctx.lib, n, k) if payload_cap is None else int(payload_cap)

    def up(v):
        return (v + 255) & ~255

    o_o = up(B)
    o_s = o_o + up(4 * B)
    o_p = o_s + up(scap + N.HSZ_SECTION_SLACK)
    o_t = o_p + up(pcap + N.HSZ_SECTION_SLACK)
    total = o_t + 16 * (T + 1)
    buf = ctx.empty(total, t.uint8)
    secs = ((buf, 0, B, None), (buf, o_o, 4 * B, t.int32),
            (buf, o_s, scap + N.HSZ_SECTION_SLACK, None),
            (buf, o_p, pcap + N.HSZ_SECTION_SLACK, None), (buf, o_t, 16 * (T + 1), t.int64))
    base = buf.data_ptr()
    ptrs = (base, base + o_o, base + o_s, base + o_p, base + o_t)
    return secs, ptrs, scap, pcap


def run_encoder(ctx: Context, params: QuantParams, launch) -> DeviceStream:
    """Run an encoder launch(widths, outliers, signs, scap, payload, pcap, toff)
    (device pointers); retry once with the exact payload size if the
    capacity policy undershot."""
    n, k = params.element_count, params.block_len
    secs, (w, o, s, p, toff), scap, pcap = new_stream_buffers(ctx, params)
    launch(w, o, s, scap, p, pcap, toff)
    ds = DeviceStream(params, *secs, ctx, scap, pcap)
    ds._ptrs = (w, o, s, p, toff)
    if pcap >= geometry(n, k)[2]:
        return ds                       # overflow impossible: stay asynchronous
    flags = ctx.read_flags()
    if flags & ~(1 << 6):
        ctx.raise_flags(flags & ~(1 << 6))
    if flags & (1 << 6):
        T = geometry(n, k)[0]
        need = int(ds.toff[2 * T + 1].item())
        secs, (w, o, s, p, toff), scap, pcap = new_stream_buffers(ctx, params, payload_cap=need)
        launch(w, o, s, scap, p, pcap, toff)
        ds = DeviceStream(params, *secs, ctx, scap, pcap)
        ds._ptrs = (w, o, s, p, toff)
        flags = ctx.read_flags()
        if flags:
            if flags & (1 << 6):
                raise CapacityExceeded("payload capacity retry failed")
            ctx.raise_flags(flags)
    return ds
