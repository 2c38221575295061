"""Homomorphic sum aggregation of several compressed streams -- the fold of
the reference's distributed-aggregation simulator (``distsim.py:80-103``,
SURVEY.md §8(f) row 1), on the GPU.

``aggregate_homomorphic(streams)`` returns the stream whose bins are the
element-wise sum of every operand's bins, built the way the reference builds
it: in the residual/outlier domain, every stream decoded once and the
accumulator re-encoded once (outliers summed in int64 and put through the
int32 guard at the end only) while the widths leave int64 headroom
(``_headroom``, distsim.py:106-110); otherwise the stream-level pairwise fold
of ``elementwise_add`` (each intermediate re-encoded and guarded).

On the device: decode stream 0 to int64 bins, decode every other stream
*into* them (``hsz_decode`` HSZ_OUT_BINS_ADD), one ``hsz_encode_bins``.  The
multi-GPU form -- every rank holds one stream, all ranks get the aggregate --
is ``sharding.Collectives.allreduce_streams``.
"""

from __future__ import annotations

import numpy as np

from . import _native as N
from .codec import _as_device_stream
from .device import DeviceStream, ptr, run_encoder, torch
from .ops import _check_params, _finish, elementwise_add

_I64_MAX = 2 ** 63 - 1


def _max_width(s) -> int:
    if isinstance(s, DeviceStream):
        w = s.widths
        return int(w.max().item()) if w.numel() else 0
    return int(s.widths.max()) if s.widths.size else 0


def _headroom(streams) -> bool:
    """distsim.py:106-110: the residual accumulation stays in int64."""
    total = sum((1 << _max_width(s)) - 1 for s in streams)
    return total <= _I64_MAX


def aggregate_homomorphic(streams, threads: int = 1, *, headroom=None):
    """Left fold of element-wise addition in the residual domain
    (distsim.py:80-96).  ``headroom`` overrides the int64-headroom test of
    distsim.py:106-110 (the multi-GPU fold of block-range slices takes it
    from the whole streams' widths, so every rank picks the same branch)."""
    streams = list(streams)
    if not streams:
        raise ValueError("need at least one stream")
    for s in streams[1:]:
        _check_params(streams[0], s)
    if len(streams) == 1:
        return streams[0]
    if headroom is None:
        headroom = _headroom(streams)
    if not headroom:
        acc = streams[0]
        for s in streams[1:]:
            acc = elementwise_add(acc, s, threads)
        return acc
    ds = [_as_device_stream(s) for s in streams]
    ctx = ds[0].ctx
    p = ds[0].params
    n, k = p.element_count, p.block_len
    bins = ctx.empty(n, torch().int64)
    bp = ptr(bins)
    for i, d in enumerate(ds):
        w, o, sg, py, toff = d.pointers()
        kind = N.HSZ_OUT_BINS if i == 0 else N.HSZ_OUT_BINS_ADD
        N.check(ctx.lib.hsz_decode(w, o, sg, py, toff, n, k, p.eps, kind, bp, ctx.err_ptr,
                                   ctx.handle), "hsz_decode")
    wsp, wsb = ctx.workspace(n, k)

    def launch(ow, oo, os_, scap, op, pcap, otoff):
        N.check(ctx.lib.hsz_encode_bins(bp, n, k, ow, oo, os_, scap, op, pcap, otoff, ctx.err_ptr,
                                        wsp, wsb, ctx.handle), "hsz_encode_bins")

    out = run_encoder(ctx, p, launch)
    return _finish(streams[0], out, "aggregate_homomorphic")


#: the reference's private name (distsim.py:80)
_aggregate_homomorphic = aggregate_homomorphic

__all__ = ["aggregate_homomorphic"]
