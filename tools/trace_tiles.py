"""Per-tile phase timeline of the compress kernel from a -DHSZ_TRACE build.

    nvcc ... -DHSZ_TRACE -o /tmp/libhsz_trace.so hsz_capi.cu
    HSZ_B200_LIB=/tmp/libhsz_trace.so python tools/trace_tiles.py
tags: 1 ticket drawn, 2 tile in smem, 3 aggregate published,
      4 previous tile placed, 5 packed
"""
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2408_11971_b200 as H  # noqa: E402
from paper_2408_11971_b200 import _native, workloads as W  # noqa: E402

x = W.config2(device="cuda").contiguous()
cfg = W.CONFIGS[2]
raw = H.RawArray(x, cfg["dims"], "f32")
lo, hi = raw.value_range()
p = H.QuantParams(cfg["rel_eps"] * (hi - lo), cfg["dims"], 32, "f32")
lib = _native.load()
for _ in range(3):
    s = H.compress(raw, p)
torch.cuda.synchronize()
lib.hsz_trace_read(None, 0, 1)
lib.hsz_trace_lookback(None)
s = H.compress(raw, p)
torch.cuda.synchronize()
lb = (ctypes.c_uint * 3)()
lib.hsz_trace_lookback(lb)
print("look-back: resolves %d  rounds/resolve %.2f  sleeps/resolve %.2f" % (lb[2], lb[0] / max(lb[2], 1), lb[1] / max(lb[2], 1)))
buf = (ctypes.c_ulonglong * (1 << 20))()
n = lib.hsz_trace_read(buf, 1 << 20, 1)
a = np.frombuffer(buf, dtype=np.uint64, count=n)
tile = (a >> 40).astype(np.int64)
tag = ((a >> 32) & 0xff).astype(np.int64)
t = (a & 0xffffffff).astype(np.int64)
t = (t - t.min()) / 1e3
nt = tile.max() + 1
T = np.full((nt, 9), np.nan)
T[tile, tag] = t
print("records", n, "tiles", nt, "span us %.1f" % np.nanmax(T))
names = {(1, 2): "load wait", (2, 3): "quant+code+scan", (3, 4): "slot/ring wait", (4, 5): "pack",
         (5, 7): "staged->placing", (7, 8): "svc resolve+copy", (3, 8): "publish->placed"}
for (a0, a1), nm in names.items():
    d = T[:, a1] - T[:, a0]
    print(f"{nm:11s} mean {np.nanmean(d):6.2f}  p50 {np.nanmedian(d):6.2f}  p90 {np.nanpercentile(d, 90):6.2f}  max {np.nanmax(d):6.2f} us")
life = T[:, 4] - T[:, 1]
print("lifetime    mean %.2f p50 %.2f" % (np.nanmean(life), np.nanmedian(life)))
for q in (0, 128, 512, 1183, 1184, 2000, 3000, 4000, 5000, nt - 1):
    if q < nt:
        print(f"tile {q:5d}: " + " ".join(f"{v:7.2f}" for v in T[q, 1:]))
# start-time histogram (10 us bins)
st = T[:, 1]
h, e = np.histogram(st, bins=np.arange(0, np.nanmax(T) + 10, 10))
print("starts per 10us:", h.tolist())
r = T[:, 5] - T[:, 4]
print("finalize by tile decile:", [round(float(np.nanmean(r[i * nt // 10:(i + 1) * nt // 10])), 2) for i in range(10)])

# service warps vs compute: when does each tile get placed (tag 8), per 5 us
pl = T[:, 8]
h, e = np.histogram(pl[~np.isnan(pl)], bins=np.arange(0, np.nanmax(T) + 5, 5))
print("resolved per 5us:", h.tolist())
h, e = np.histogram(T[:, 1][~np.isnan(T[:, 1])], bins=np.arange(0, np.nanmax(T) + 5, 5))
print("started per 5us:", h.tolist())
print("first start %.2f  last start %.2f  last pack %.2f  last resolve %.2f" % (
    np.nanmin(T[:, 1]), np.nanmax(T[:, 1]), np.nanmax(T[:, 4]), np.nanmax(T[:, 8])))
