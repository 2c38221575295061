"""Per-tile phase timeline of the scalar_mul kernel (-DHSZ_TRACE build).
tags: 1 input tile ready, 2 widths scanned, 3 decoded + rescaled, 4 coded +
scanned + slot free, 5 packed; placement warp: 7 resolve start, 8 copied out"""
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2408_11971_b200 as H  # noqa: E402
from paper_2408_11971_b200 import _native, workloads as W  # noqa: E402

CONFIG = int(sys.argv[1]) if len(sys.argv) > 1 else 2
x = torch.from_numpy(W.field(CONFIG)).cuda().contiguous()
cfg = W.CONFIGS[CONFIG]
raw = H.RawArray(x, cfg["dims"], "f32")
lo, hi = raw.value_range()
p = H.QuantParams(cfg["rel_eps"] * (hi - lo), cfg["dims"], 32, "f32")
s = H.scalar_add(H.negate(H.compress(raw, p)), cfg["sadd"])
lib = _native.load()
for _ in range(3):
    z = H.scalar_mul(s, cfg["smul"])
torch.cuda.synchronize()
lib.hsz_trace_read(None, 0, 1)
lib.hsz_trace_lookback(None)
z = H.scalar_mul(s, cfg["smul"])
torch.cuda.synchronize()
lb = (ctypes.c_uint * 3)()
lib.hsz_trace_lookback(lb)
print("look-back: rounds %d sleeps %d resolves %d -> %.2f rounds, %.2f sleeps per resolve" %
      (lb[0], lb[1], lb[2], lb[0] / max(lb[2], 1), lb[1] / max(lb[2], 1)))
buf = (ctypes.c_ulonglong * (1 << 20))()
n = lib.hsz_trace_read(buf, 1 << 20, 1)
a = np.frombuffer(buf, dtype=np.uint64, count=n)
tile = (a >> 40).astype(np.int64)
tag = ((a >> 32) & 0xff).astype(np.int64)
t = (a & 0xffffffff).astype(np.int64)
t = (t - t.min()) / 1e3
keep = tile < (1 << 23)
tile, tag, t = tile[keep], tag[keep], t[keep]
nt = tile.max() + 1
T = np.full((nt, 9), np.nan)
T[tile, tag] = t
print("records", n, "tiles", nt, "span us %.1f" % np.nanmax(T))
for (a0, a1), nm in {(1, 2): "widths scan", (2, 3): "decode+rescale", (3, 4): "code+scan+slot",
                     (4, 5): "pack", (5, 7): "staged->resolve", (7, 8): "resolve+copy"}.items():
    d = T[:, a1] - T[:, a0]
    print(f"{nm:16s} mean {np.nanmean(d):6.2f}  p50 {np.nanmedian(d):6.2f}  p90 {np.nanpercentile(d, 90):6.2f} us")
st = np.sort(T[:, 1][~np.isnan(T[:, 1])])
print("iteration gap (start of consecutive tiles, same CTA unknown) -- tile starts per 10 us:",
      np.histogram(st, bins=np.arange(0, st.max() + 10, 10))[0].tolist())
