"""Phase timing of the compress kernel from a -DHSZ_TRACE build.
    HSZ_B200_LIB=.../libhsz_trace.so python tools/trace_encode.py"""
import ctypes
import os
import sys
from collections import defaultdict

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
for _ in range(2):
    s = H.compress(raw, p)
torch.cuda.synchronize()
lib.hsz_trace_read(None, 0, 1)
s = H.compress(raw, p)
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * (1 << 20))()
n = lib.hsz_trace_read(buf, 1 << 20, 1)
a = np.frombuffer(buf, dtype=np.uint64, count=n)
cta = (a >> 48).astype(np.int64)
tag = ((a >> 40) & 0xff).astype(np.int64)
t = (a & ((1 << 40) - 1)).astype(np.int64)
t0 = t.min()
print("records", n, "span us", (t.max() - t0) / 1e3)
# per CTA, consecutive tag pairs
dur = defaultdict(list)
order = np.lexsort((t, cta))
cta, tag, t = cta[order], tag[order], t[order]
for i in range(len(t) - 1):
    if cta[i] == cta[i + 1]:
        dur[(tag[i], tag[i + 1])].append(t[i + 1] - t[i])
for k in sorted(dur):
    v = np.array(dur[k])
    print(f"{k[0]}->{k[1]}: n={len(v):6d} mean={v.mean()/1e3:7.2f}us p50={np.median(v)/1e3:7.2f} p90={np.percentile(v,90)/1e3:7.2f} total={v.sum()/1e3/592:8.2f}us/CTA")
first = defaultdict(lambda: 1 << 62)
last = defaultdict(int)
for c, tt in zip(cta, t):
    first[c] = min(first[c], tt)
    last[c] = max(last[c], tt)
st = np.array([first[c] - t0 for c in first]) / 1e3
en = np.array([last[c] - t0 for c in last]) / 1e3
print("CTA start: p50 %.1f max %.1f us;  end: min %.1f p50 %.1f max %.1f us" % (np.median(st), st.max(), en.min(), np.median(en), en.max()))
