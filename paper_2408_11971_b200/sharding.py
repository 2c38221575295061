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
``allreduce_streams``: one all_gather of the serialized (compressed) streams,
then the residual-domain fold of distsim.py:80-103 (``distsim.py`` here).

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


class Collectives:
    """The three collectives over a torch.distributed process group."""

    def __init__(self, group=None, device=None):
        import torch
        import torch.distributed as dist

        self.dist = dist
        self.torch = torch
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        backend = dist.get_backend(group)
        if device is None:
            device = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" \
                else torch.device("cpu")
        self.device = device

    def global_range(self, lo: float, hi: float):
        """C1: allreduce MIN over (lo, -hi) in float64 (exact)."""
        t = self.torch.tensor([lo, -hi], dtype=self.torch.float64, device=self.device)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MIN, group=self.group)
        v = t.cpu().tolist()
        return float(v[0]), float(-v[1])

    def _allgather_i64(self, vals):
        t = self.torch.tensor([int(v) for v in vals], dtype=self.torch.int64, device=self.device)
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
        """C3: allgather of exact (S, Q) as 64-bit limbs, exact host sum."""
        limbs = _to_limbs(S, Q)
        rows = self._allgather_i64(limbs)
        tot_s = tot_q = 0
        for r in rows:
            s, q = _from_limbs(r)
            tot_s += s
            tot_q += q
        return tot_s, tot_q

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
        residual-domain fold of distsim.py:80-103, on this rank's GPU by
        default; `fold` overrides it, e.g. with the CPU oracle in tests)."""
        streams = self.gather_streams(stream)
        if fold is None:
            from .distsim import aggregate_homomorphic as fold
        return fold(streams)

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
        t = self.torch.tensor([value], dtype=self.torch.float64, device=self.device)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX, group=self.group)
        return float(t.item())


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
