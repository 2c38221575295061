"""Host time of the pieces of one H.compress call (median of 300, no sync
inside the loop): where the launch latency after the value-range sync goes.

    python tools/host_compress_parts.py
"""
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2408_11971_b200 as H  # noqa: E402
from paper_2408_11971_b200 import codec as C  # noqa: E402
from paper_2408_11971_b200 import device as D  # noqa: E402
from paper_2408_11971_b200 import workloads as W  # noqa: E402

cfg = W.CONFIGS[2]
x = torch.from_numpy(W.config2()).cuda()
raw = H.RawArray(x, cfg["dims"], "f32")
lo, hi = raw.value_range()
p = H.QuantParams(cfg["rel_eps"] * (hi - lo), cfg["dims"], 32, "f32")
ctx = D.context()
n = p.element_count


def t_of(fn, reps=300):
    for _ in range(20):
        fn()
    torch.cuda.synchronize()
    ts = []
    for i in range(reps):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
        if i % 30 == 29:
            torch.cuda.synchronize()
    return round(1e6 * statistics.median(ts), 2)


rows = {
    "H.compress": lambda: H.compress(raw, p),
    "compress_device": lambda: C.compress_device(x, p, ctx),
    "_check_geometry": lambda: C._check_geometry(raw, p),
    "context()": lambda: D.context(),
    "raw.device_values": lambda: raw.device_values(ctx),
    "ctx.workspace": lambda: ctx.workspace(n, 32),
    "new_stream_buffers": lambda: D.new_stream_buffers(ctx, p),
    "geometry(n,k)": lambda: D.geometry(n, 32),
    "p.element_count": lambda: p.element_count,
}
for k, fn in rows.items():
    print(f"{k:24s} {t_of(fn):8.2f} us")
