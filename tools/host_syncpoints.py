"""Host time of each public call of the chain (median of 200): the
synchronising calls (value range, mean, variance) include their kernel; the
rest are launch-only.  Together with tools/time_ops.py's kernel times this
says how much host time sits on the GPU's critical path at each sync point.

    python tools/host_syncpoints.py
"""
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2408_11971_b200 as H  # noqa: E402
from paper_2408_11971_b200 import workloads as W  # noqa: E402

cfg = W.CONFIGS[2]
x = torch.from_numpy(W.config2()).cuda()
raw = H.RawArray(x, cfg["dims"], "f32")
lo, hi = raw.value_range()
eps = cfg["rel_eps"] * (hi - lo)
p = H.QuantParams(eps, cfg["dims"], 32, "f32")
s = H.compress(raw, p)
z = H.scalar_mul(H.scalar_add(H.negate(s), cfg["sadd"]), cfg["smul"])
torch.cuda.synchronize()


def t_of(fn, reps=200):
    ts = []
    for _ in range(reps + 10):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    torch.cuda.synchronize()
    return round(1e6 * statistics.median(ts[10:]), 1)


rows = {
    "RawArray(x) [minmax kernel + sync]": lambda: H.RawArray(x, cfg["dims"], "f32"),
    "QuantParams(...)": lambda: H.QuantParams(eps, cfg["dims"], 32, "f32"),
    "compress [launch]": lambda: H.compress(raw, p),
    "negate [launch]": lambda: H.negate(s),
    "scalar_add [launch]": lambda: H.scalar_add(s, cfg["sadd"]),
    "scalar_mul [launch]": lambda: H.scalar_mul(s, cfg["smul"]),
    "mean [kernel + sync]": lambda: H.mean(z),
    "variance [kernel + sync]": lambda: H.variance(z),
    "decompress [launch]": lambda: H.decompress(z),
}
print(json.dumps({k: t_of(fn) for k, fn in rows.items()}, indent=1))
