"""Multi-GPU partitioning of one field by contiguous block ranges.

One process per GPU (torch.distributed, NCCL over NVLink/NVSwitch; gloo for
the CPU tests).  Blocks are independent and byte-aligned (FORMAT.md:39-40),
so each rank compresses / transforms its own block range with no data-path
exchange.  Only three tiny, latency-bound collectives exist:

* C1 ``global_range`` -- allreduce MIN/MAX of the local value range, so every
  rank resolves the identical relative eps (codec.py:96-99);
* C2 ``global_offsets`` -- allgather of per-shard (sign bytes, payload bytes)
  and an exclusive scan: where each shard's sections start in the global
  stream (widths/outliers start at the shard's first block);
* C3 ``global_moments`` -- allgather of the exact per-shard (S, Q) limbs and
  an exact host sum, so mean / variance are bit-identical for any GPU count.

A second pattern -- every rank holds a whole stream of the same geometry
(ensemble members, time steps) and all want their sum -- is
``allreduce_streams``: a reduce-scatter over tile-aligned block ranges (one
all_to_all of compressed slices, each rank folds its range with the
residual-domain fold of distsim.py:80-103) and an all_gather of the
compressed partial sums.  ``gather_streams`` (every rank gets every stream)
stays for callers that want the operands themselves.

The shard's sections, concatenated in rank order at the C2 offsets, are
byte-identical to the single-GPU stream of the whole field (tested in
tests/test_sharding_gloo.py and tests/test_gpu_sharding.py).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


def block_range(nblocks: int, rank: int, world: int):
    """Contiguous, balanced block range [b0, b1) of `rank`."""
    base, extra = divmod(nblocks, world)
    b0 = rank * base + min(rank, extra)
    b1 = b0 + base + (1 if rank < extra else 0)
    return b0, b1


def element_range(n: int, block_len: int, rank: int, world: int):
    nb = -(-n // block_len)
    b0, b1 = block_range(nb, rank, world)
    return b0 * block_len, min(b1 * block_len, n)


def exclusive_scan(values):
    out, acc = [], 0
    for v in values:
        out.append(acc)
        acc += int(v)
    return out, acc


@dataclass
class ShardLayout:
    """Where one shard's sections sit inside the global stream."""

    rank: int
    block0: int
    sign_offset: int
    payload_offset: int
    sign_total: int
    payload_total: int


class HostAllGather:
    """Node-local all-gather of a few int64 words per rank through a shared
    memory segment (C ABI ``hsz_hostcoll_allgather``): the small exchanges of
    the chain (C1-C3) carry host scalars, so between the processes of one
    node they need no device round trip.  Raises RuntimeError at setup when
    the ranks are not on one host."""

    MAX_VALS = 40

    def __init__(self, dist, group, rank: int, world: int, timeout_s: float = 300.0):
        import ctypes
        import mmap
        import os
        import socket
        import tempfile
        import uuid

        from . import _native as N

        self.lib = N.load()
        self.rank, self.world, self.timeout = rank, world, float(timeout_s)
        info = [None] * world
        dist.all_gather_object(info, (socket.gethostname(), uuid.uuid4().hex), group=group)
        if len({h for h, _ in info}) != 1:
            raise RuntimeError("ranks span several hosts")
        root = "/dev/shm" if os.path.isdir("/dev/shm") else tempfile.gettempdir()
        path = os.path.join(root, f"hsz_coll_{info[0][1]}")
        size = int(self.lib.hsz_hostcoll_bytes(world))
        token = info[0][1].encode()            # rank 0 writes it, every rank must read it back
        ok, err = True, ""
        if rank == 0:
            try:
                fd = os.open(path, os.O_CREAT | os.O_EXCL | os.O_RDWR, 0o600)
                os.ftruncate(fd, size + 64)
                os.pwrite(fd, token, size)
                os.close(fd)
            except OSError as e:
                ok, err = False, repr(e)
        dist.barrier(group=group)
        mm = None
        if ok:
            # a shared hostname does not prove a shared /dev/shm (private IPC
            # namespaces, pods with equal hostnames): map the segment and
            # check rank 0's token; every rank then agrees on the outcome
            try:
                fd = os.open(path, os.O_RDWR)
                try:
                    mm = mmap.mmap(fd, size + 64)
                finally:
                    os.close(fd)
                ok = mm[size:size + len(token)] == token
                if not ok:
                    err = "token mismatch"
            except OSError as e:
                ok, err = False, repr(e)
        votes = [None] * world
        dist.all_gather_object(votes, (ok, err), group=group)
        if rank == 0:
            try:
                os.unlink(path)          # the mappings stay; nothing left behind
            except OSError:
                pass
        bad = [(r, e) for r, (v, e) in enumerate(votes) if not v]
        if bad:
            if mm is not None:
                mm.close()
            raise RuntimeError(f"node-local shared memory unusable on rank {bad[0][0]}: {bad[0][1]}")
        self._mm = mm
        self._buf = (ctypes.c_char * size).from_buffer(self._mm)
        self._addr = ctypes.addressof(self._buf)
        self._round = 0
        self._vals = np.zeros(self.MAX_VALS, dtype=np.int64)
        self._out = np.zeros(world * self.MAX_VALS, dtype=np.int64)

    def __call__(self, vals):
        nv = len(vals)
        self._vals[:nv] = vals
        self._round += 1
        rc = self.lib.hsz_hostcoll_allgather(self._addr, self.rank, self.world, self._round,
                                             self._vals.ctypes.data, nv, self._out.ctypes.data,
                                             self.timeout)
        if rc != 0:
            raise RuntimeError(f"host all-gather round {self._round} failed ({rc}): a peer "
                               "did not publish in time")
        return self._out[:self.world * nv].reshape(self.world, nv).tolist()


def _f2i(v: float) -> int:
    import struct

    return struct.unpack("<q", struct.pack("<d", float(v)))[0]


def _i2f(v: int) -> float:
    import struct

    return struct.unpack("<d", struct.pack("<q", int(v)))[0]


class Collectives:
    """The three collectives over a torch.distributed process group.

    By default every exchange runs on the process group (NCCL on the GPU
    path, as north_star names them: C1 an allreduce MIN, C2 an allgather of
    the shard byte counts, C3 an allreduce SUM of int64 partial sums).
    ``host_shm=True`` (or ``HSZ_HOSTCOLL=1``) moves the small host-scalar
    exchanges to a node-local shared-memory all-gather (4-8 us instead of
    44-57 us per NCCL round trip, profiles/r1e_coll_latency.json) when every
    rank can map the same segment; setup failure on any rank makes every
    rank fall back to the process group together.  Bulk data always moves
    over the process group."""

    def __init__(self, group=None, device=None, host_shm=None):
        import os

        import torch
        import torch.distributed as dist

        self.dist = dist
        self.torch = torch
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.backend = dist.get_backend(group)
        if device is None:
            device = torch.device("cuda", torch.cuda.current_device()) if self.backend == "nccl" \
                else torch.device("cpu")
        self.device = device
        if host_shm is None:
            host_shm = os.environ.get("HSZ_HOSTCOLL", "0") == "1"
        self._hc = None
        if host_shm:
            try:
                self._hc = HostAllGather(dist, group, self.rank, self.world)
            except RuntimeError:
                self._hc = None          # agreed on every rank: process group only

    @property
    def host_shm(self) -> bool:
        return self._hc is not None

    def global_range(self, lo: float, hi: float):
        """C1: MIN over (lo, -hi) in float64 (exact)."""
        if self._hc is not None:
            rows = self._hc([_f2i(lo), _f2i(-hi)])
            return min(_i2f(r[0]) for r in rows), -min(_i2f(r[1]) for r in rows)
        t = self.torch.tensor([lo, -hi], dtype=self.torch.float64, device=self.device)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MIN, group=self.group)
        v = t.cpu().tolist()
        return float(v[0]), float(-v[1])

    def _allgather_i64(self, vals):
        vals = [int(v) for v in vals]
        if self._hc is not None and len(vals) <= HostAllGather.MAX_VALS:
            return self._hc(vals)
        t = self.torch.tensor(vals, dtype=self.torch.int64, device=self.device)
        if self.backend == "nccl":
            out = self.torch.empty(self.world * len(vals), dtype=self.torch.int64,
                                   device=self.device)
            self.dist.all_gather_into_tensor(out, t, group=self.group)
            flat = out.cpu().tolist()
            return [flat[i * len(vals):(i + 1) * len(vals)] for i in range(self.world)]
        out = [self.torch.empty_like(t) for _ in range(self.world)]
        self.dist.all_gather(out, t, group=self.group)
        return [[int(x) for x in o.cpu().tolist()] for o in out]

    def global_offsets(self, block0: int, sign_bytes: int, payload_bytes: int) -> ShardLayout:
        """C2: allgather of the shard byte counts, exclusive scan."""
        rows = self._allgather_i64([block0, sign_bytes, payload_bytes])
        so, st = exclusive_scan(r[1] for r in rows)
        po, pt = exclusive_scan(r[2] for r in rows)
        return ShardLayout(self.rank, block0, so[self.rank], po[self.rank], st, pt)

    def global_moments(self, S: int, Q: int):
        """C3: exact global (S, Q).  On the process group: ONE allreduce SUM
        of int64 partial sums -- S (int128) and Q (uint192) as ten 32-bit
        chunks, so the sum cannot overflow for any world size below 2^31 and
        the recombined totals are exact; on the shared-memory path an
        allgather of 64-bit limbs and an exact host sum."""
        if self._hc is not None:
            rows = self._hc(_to_limbs(S, Q))
            tot_s = tot_q = 0
            for r in rows:
                s, q = _from_limbs(r)
                tot_s += s
                tot_q += q
            return tot_s, tot_q
        t = self.torch.tensor(_to_chunks(S, Q), dtype=self.torch.int64, device=self.device)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM, group=self.group)
        return _from_chunks(t.cpu().tolist())

    def global_offsets_many(self, block0: int, sizes):
        """C2 for several streams of this rank's shard in one exchange:
        `sizes` = [(sign bytes, payload bytes), ...] -> [ShardLayout, ...]."""
        sizes = [(int(a), int(b)) for a, b in sizes]
        rows = self._allgather_i64([block0] + [v for sp in sizes for v in sp])
        lays = []
        for j in range(len(sizes)):
            so, st = exclusive_scan(r[1 + 2 * j] for r in rows)
            po, pt = exclusive_scan(r[2 + 2 * j] for r in rows)
            lays.append(ShardLayout(self.rank, block0, so[self.rank], po[self.rank], st, pt))
        return lays

    def global_moments_offsets(self, S: int, Q: int, block0: int, sizes):
        """C3 with C2 riding along: the exact (S, Q) totals and, for every
        stream in `sizes` ((sign bytes, payload bytes) of this rank's shard),
        its ShardLayout -- one exchange instead of one per collective, at a
        point where the host has synchronised anyway (a moment result)."""
        sizes = [(int(a), int(b)) for a, b in sizes]
        rows = self._allgather_i64(_to_limbs(S, Q) + [block0] + [v for sp in sizes for v in sp])
        tot_s = tot_q = 0
        for r in rows:
            s, q = _from_limbs(r[:5])
            tot_s += s
            tot_q += q
        lays = []
        for j in range(len(sizes)):
            so, st = exclusive_scan(r[6 + 2 * j] for r in rows)
            po, pt = exclusive_scan(r[7 + 2 * j] for r in rows)
            lays.append(ShardLayout(self.rank, block0, so[self.rank], po[self.rank], st, pt))
        return tot_s, tot_q, lays

    # -- reduce compressed streams (distsim.py:80-103 across ranks) ---------
    def gather_streams(self, stream):
        """Every rank's stream (same params) on every rank, in rank order, as
        host CompressedStreams: the serialized bytes (FORMAT.md) of each
        rank travel through one padded all_gather -- compressed, so a
        fraction of the raw field's size."""
        from .device import DeviceStream
        from .model import deserialize, serialize

        host = stream.to_host() if isinstance(stream, DeviceStream) else stream
        blob = serialize(host)
        sizes = [r[0] for r in self._allgather_i64([len(blob)])]
        t = self.torch
        buf = t.zeros(max(sizes), dtype=t.uint8)
        buf[:len(blob)] = t.frombuffer(bytearray(blob), dtype=t.uint8)
        buf = buf.to(self.device)
        out = [t.empty_like(buf) for _ in range(self.world)]
        self.dist.all_gather(out, buf, group=self.group)
        return [deserialize(bytes(o[:sz].cpu().numpy().tobytes())) for o, sz in zip(out, sizes)]

    def allreduce_streams(self, stream, fold=None):
        """Every rank gets the homomorphic sum of all ranks' streams (the
        residual-domain fold of distsim.py:80-103 across ranks), as a
        reduce-scatter over tile-aligned block ranges followed by an
        all-gather of the compressed partial sums:

        1. every rank cuts its stream into ``world`` block-range slices at
           tile boundaries (offsets from the tile-offset cache: a block range
           of a stream is itself a stream, FORMAT.md blocks being
           byte-aligned);
        2. one ``all_to_all``: rank r receives every rank's slice r;
        3. rank r folds the ``world`` slices of its range on its GPU (``fold``
           overrides the fold, e.g. with the CPU oracle in tests).  The
           int64-headroom branch of distsim.py:106-110 is chosen from the
           whole streams' widths (allgathered), so every rank takes the
           branch the single-process fold takes;
        4. errors are agreed across ranks -- the first failing fold step,
           then the reference's precedence (errors.raise_for_flags) -- so
           every rank raises what the single-process fold raises;
        5. one ``all_gather`` of the partial sums; concatenated in rank order
           they are the aggregate stream, byte-identical to the single-process
           fold.

        Per rank: (world-1)/world of one stream out and in, plus the
        compressed result, and one stream's worth of fold work."""
        from .device import DeviceStream
        from .errors import ParamsMismatch

        t = self.torch
        world, me = self.world, self.rank
        on_dev = isinstance(stream, DeviceStream)
        p = stream.params
        n, k, B = p.element_count, p.block_len, p.block_count
        cuts, so, po, maxw = _cut_points(stream, world)
        # exchange: params digest, max width, and the bytes of every slice
        rows = self._allgather_i64([_params_digest(p), maxw]
                                   + [so[j + 1] - so[j] for j in range(world)]
                                   + [po[j + 1] - po[j] for j in range(world)])
        if any(r[0] != rows[0][0] for r in rows):
            raise ParamsMismatch("operand params differ across ranks")
        headroom = sum((1 << r[1]) - 1 for r in rows) <= (1 << 63) - 1

        # 1-2: slices out, my range's slices in
        secs = _section_bytes(stream)
        out_parts, in_splits = [], []
        for j in range(world):
            b0, b1 = cuts[j], cuts[j + 1]
            out_parts += [secs[0][b0:b1], secs[1][4 * b0:4 * b1], secs[2][so[j]:so[j + 1]],
                          secs[3][po[j]:po[j + 1]]]
            in_splits.append(5 * (b1 - b0) + (so[j + 1] - so[j]) + (po[j + 1] - po[j]))
        send = t.cat(out_parts).to(self.device)
        mb0, mb1 = cuts[me], cuts[me + 1]
        nb = mb1 - mb0
        sizes = [(rows[i][2 + me], rows[i][2 + world + me]) for i in range(world)]
        out_splits = [5 * nb + ss + ps for ss, ps in sizes]
        recv = t.empty(sum(out_splits), dtype=t.uint8, device=self.device)
        self.dist.all_to_all_single(recv, send, out_splits, in_splits, group=self.group)

        # 3-4: fold my range
        ctx = stream.ctx if on_dev else None
        part = None
        if nb:
            from .model import QuantParams

            pr = QuantParams(p.eps, (min(mb1 * k, n) - mb0 * k,), k, p.dtype)
            subs, pos = [], 0
            for ss, ps in sizes:
                w, o, sg, py = _split(recv, pos, (nb, 4 * nb, ss, ps))
                pos += 5 * nb + ss + ps
                subs.append(_make_stream(pr, w, o, sg, py, ctx))
        if fold is not None:
            part = self._agreed(lambda: fold(subs) if nb else None, ctx)
        elif headroom:
            from .distsim import aggregate_homomorphic

            part = self._agreed(
                lambda: aggregate_homomorphic(subs, headroom=True) if nb else None, ctx)
        else:
            from .ops import elementwise_add

            part = subs[0] if nb else None
            for i in range(1, world):
                part = self._agreed(lambda: elementwise_add(part, subs[i]) if nb else None, ctx)

        # 5: partial sums to everyone, concatenated in rank order
        if nb:
            rsec = _section_bytes(part)
            blob = t.cat(rsec).to(self.device)
            mine = [int(rsec[2].numel()), int(rsec[3].numel())]
        else:
            blob = t.empty(0, dtype=t.uint8, device=self.device)
            mine = [0, 0]
        rrows = self._allgather_i64([blob.numel()] + mine)
        top = max(r[0] for r in rrows)
        padded = t.zeros(max(top, 1), dtype=t.uint8, device=self.device)
        padded[:blob.numel()] = blob
        got = [t.empty_like(padded) for _ in range(world)]
        self.dist.all_gather(got, padded, group=self.group)
        cols = [[], [], [], []]
        for i in range(world):
            nbi = cuts[i + 1] - cuts[i]
            for c, x in zip(cols, _split(got[i], 0, (nbi, 4 * nbi, rrows[i][1], rrows[i][2]))):
                c.append(x)
        full = [t.cat(c) for c in cols]
        return _make_stream(p, *full, ctx)

    def _agreed(self, step, ctx):
        """Run one fold step and agree on its outcome across ranks: if any
        rank failed, every rank raises the error of highest precedence."""
        err, res = None, None
        try:
            res = step()
            if ctx is not None:
                flags = ctx.read_flags()
                if flags:
                    ctx.raise_flags(flags, "allreduce_streams")
        except Exception as e:        # any failure still takes part in the agreement
            err = e
        code = 0 if err is None else _precedence(err)
        codes = [r[0] for r in self._allgather_i64([code])]
        bad = [c for c in codes if c]
        if bad:
            c = min(bad)
            if err is not None and code == c:
                raise err
            raise _EXC_BY_CODE[c](f"allreduce_streams: fold failed on rank {codes.index(c)}")
        return res

    def write_sharded(self, path, params, layout: ShardLayout, stream):
        """Every rank writes its shard's sections straight into one ``.hsz``
        file at the global offsets (FORMAT.md; C2 layout) -- no gather.
        `params` = the whole field's QuantParams, `stream` = this rank's shard
        (host or device)."""
        import os

        from .device import DeviceStream
        from .model import header_bytes

        host = stream.to_host() if isinstance(stream, DeviceStream) else stream
        hdr = header_bytes(params)
        h, B = len(hdr), params.block_count
        total = h + 5 * B + layout.sign_total + layout.payload_total
        if self.rank == 0:
            with open(path, "wb") as f:
                f.truncate(total)
                f.write(hdr)
        self.barrier()
        fd = os.open(path, os.O_WRONLY)
        try:
            b0 = layout.block0
            os.pwrite(fd, np.asarray(host.widths, dtype=np.uint8).tobytes(), h + b0)
            os.pwrite(fd, np.asarray(host.outliers, dtype="<i4").tobytes(), h + B + 4 * b0)
            if len(host.sign_planes):
                os.pwrite(fd, bytes(host.sign_planes), h + 5 * B + layout.sign_offset)
            if len(host.payload):
                os.pwrite(fd, bytes(host.payload),
                          h + 5 * B + layout.sign_total + layout.payload_offset)
        finally:
            os.close(fd)
        self.barrier()
        return total

    def barrier(self):
        self.dist.barrier(group=self.group)

    def max_over_ranks(self, value: float) -> float:
        if self._hc is not None:
            return max(_i2f(r[0]) for r in self._hc([_f2i(value)]))
        t = self.torch.tensor([value], dtype=self.torch.float64, device=self.device)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX, group=self.group)
        return float(t.item())


def _to_chunks(S: int, Q: int):
    """S (signed, two's complement mod 2^128) and Q (unsigned, < 2^192) as ten
    non-negative 32-bit chunks (int64 slots: summable over < 2^31 ranks)."""
    s = S & ((1 << 128) - 1)
    return [(s >> (32 * k)) & 0xFFFFFFFF for k in range(4)] + \
        [(Q >> (32 * k)) & 0xFFFFFFFF for k in range(6)]


def _from_chunks(chunks):
    """Sum of chunk vectors -> exact (S, Q) (S wrapped back to signed 128-bit)."""
    c = [int(v) for v in chunks]
    s = sum(c[k] << (32 * k) for k in range(4)) & ((1 << 128) - 1)
    if s >= 1 << 127:
        s -= 1 << 128
    q = sum(c[4 + k] << (32 * k) for k in range(6))
    return s, q


def _to_limbs(S: int, Q: int):
    """S (signed, < 2^127) and Q (unsigned, < 2^192) -> 5 int64 limbs."""
    m = (1 << 64) - 1
    s = S & ((1 << 128) - 1)
    limbs = [s & m, s >> 64, Q & m, (Q >> 64) & m, Q >> 128]
    return [v - (1 << 64) if v >= (1 << 63) else v for v in limbs]


def _from_limbs(limbs):
    u = [int(v) & ((1 << 64) - 1) for v in limbs]
    S = u[0] | (u[1] << 64)
    if S >= 1 << 127:
        S -= 1 << 128
    Q = u[2] | (u[3] << 64) | (u[4] << 128)
    return S, Q


# -- block-range slices of whole streams (allreduce_streams) -------------------
_TILE_BLOCKS = 128    # blocks per tile of the device tile-offset cache (hsz_b200.h)


def tile_block_range(nblocks: int, rank: int, world: int):
    """Contiguous block range [b0, b1) of `rank`, cut at tile boundaries."""
    T = -(-nblocks // _TILE_BLOCKS)
    t0, t1 = block_range(T, rank, world)
    return min(t0 * _TILE_BLOCKS, nblocks), min(t1 * _TILE_BLOCKS, nblocks)


def _cut_points(stream, world):
    """Block, sign-byte and payload-byte offsets of the world+1 cut points of
    `stream`, and its maximum width.  Device streams read them from the
    tile-offset cache (one small copy); host streams from the section sizes."""
    from .device import DeviceStream

    B = stream.params.block_count
    cuts = [tile_block_range(B, j, world)[0] for j in range(world)] + [B]
    if isinstance(stream, DeviceStream):
        t = __import__("torch")
        tiles = [-(-b // _TILE_BLOCKS) for b in cuts]
        idx = t.tensor([2 * x for x in tiles] + [2 * x + 1 for x in tiles], dtype=t.int64,
                       device=stream.ctx.device)
        sel = stream.toff.index_select(0, idx)
        mw = stream.widths.max().to(t.int64).reshape(1)
        sel_h, mw_h = stream.ctx.fetch_checked([sel, mw], "allreduce_streams")
        so = [int(v) for v in sel_h[:world + 1]]
        po = [int(v) for v in sel_h[world + 1:]]
        return cuts, so, po, int(mw_h[0])
    cs = np.concatenate([[0], np.cumsum(stream.sign_sizes(), dtype=np.int64)])
    cp = np.concatenate([[0], np.cumsum(stream.payload_sizes(), dtype=np.int64)])
    maxw = int(stream.widths.max()) if B else 0
    return cuts, [int(cs[b]) for b in cuts], [int(cp[b]) for b in cuts], maxw


def _section_bytes(stream):
    """The four sections of a stream as flat uint8 torch tensors (device
    views for a DeviceStream, CPU tensors for a host stream)."""
    import torch as t

    from .device import DeviceStream

    if isinstance(stream, DeviceStream):
        sb, pb = stream.totals()
        return [stream.widths, stream.outliers.view(t.uint8), stream.signs[:sb],
                stream.payload[:pb]]
    return [t.from_numpy(np.ascontiguousarray(stream.widths, dtype=np.uint8).copy()),
            t.from_numpy(np.ascontiguousarray(stream.outliers, dtype="<i4").view(np.uint8).copy()),
            t.from_numpy(np.frombuffer(stream.sign_planes, dtype=np.uint8).copy()),
            t.from_numpy(np.frombuffer(stream.payload, dtype=np.uint8).copy())]


def _split(buf, pos, lens):
    out = []
    for ln in lens:
        out.append(buf[pos:pos + ln])
        pos += ln
    return out


def _make_stream(params, w, o, sg, py, ctx):
    """A stream of `params` from its four uint8 sections: on `ctx`'s device
    (ctx given) or on the host."""
    if ctx is not None:
        from .device import DeviceStream

        dev = ctx.device
        return DeviceStream.from_sections(params, w.to(dev), o.to(dev), sg.to(dev), py.to(dev),
                                          ctx)
    from .model import CompressedStream

    return CompressedStream(params, w.cpu().numpy(), o.cpu().numpy().view("<i4"),
                            sg.cpu().numpy().tobytes(), py.cpu().numpy().tobytes())


def _params_digest(p) -> int:
    import hashlib

    key = repr((float(p.eps).hex(), tuple(p.dims), int(p.block_len), p.dtype)).encode()
    return int.from_bytes(hashlib.sha1(key).digest()[:8], "little", signed=True)


def _precedence(err) -> int:
    """errors.raise_for_flags order (1 = highest); 7 = a failure outside the
    reference's error classes (CUDA RuntimeError, OverflowError, ...)."""
    from .errors import (CapacityExceeded, GeometryMismatch, HoszpError, OutlierOverflow,
                         QuantOverflow)

    for code, cls in ((2, GeometryMismatch), (3, QuantOverflow), (4, OutlierOverflow),
                      (5, CapacityExceeded)):
        if isinstance(err, cls):
            return code
    if isinstance(err, ValueError):
        return 1
    return 6 if isinstance(err, HoszpError) else 7


def _exc_by_code():
    from .errors import (CapacityExceeded, GeometryMismatch, HoszpError, OutlierOverflow,
                         QuantOverflow)

    return {1: ValueError, 2: GeometryMismatch, 3: QuantOverflow, 4: OutlierOverflow,
            5: CapacityExceeded, 6: HoszpError, 7: RuntimeError}


class _LazyCodes(dict):
    def __missing__(self, code):
        self.update(_exc_by_code())
        return dict.__getitem__(self, code)


_EXC_BY_CODE = _LazyCodes()


def assemble(params, layouts, shards):
    """Concatenate per-shard host sections (widths, outliers, signs, payload),
    given in rank order with their layouts, into one global CompressedStream."""
    from .model import CompressedStream

    order = sorted(range(len(layouts)), key=lambda i: layouts[i].rank)
    widths = np.concatenate([np.asarray(shards[i][0], dtype=np.uint8) for i in order])
    outl = np.concatenate([np.asarray(shards[i][1], dtype=np.int64) for i in order])
    signs = b"".join(bytes(shards[i][2]) for i in order)
    payload = b"".join(bytes(shards[i][3]) for i in order)
    for i in order:
        L = layouts[i]
        assert L.sign_offset == sum(len(shards[j][2]) for j in order if layouts[j].rank < L.rank)
    return CompressedStream(params, widths, outl, signs, payload)
