"""Host-side (launch) latency of each public-API call, no synchronisation:
the wall time the Python layer spends per call, which the GPU sees as idle
time right after a synchronising call (value range, mean, variance)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2408_11971_b200 as H  # noqa: E402
from paper_2408_11971_b200 import ops as O  # noqa: E402
from paper_2408_11971_b200 import workloads as W  # noqa: E402

cfg = W.CONFIGS[2]
x = torch.from_numpy(W.config2()).cuda()
raw = H.RawArray(x, cfg["dims"], "f32")
lo, hi = raw.value_range()
p = H.QuantParams(cfg["rel_eps"] * (hi - lo), cfg["dims"], 32, "f32")
s = H.compress(raw, p)
z = H.scalar_mul(H.scalar_add(H.negate(s), 3.5), -1.25)
torch.cuda.synchronize()
fns = {
    "RawArray+range(sync)": lambda: H.RawArray(x, cfg["dims"], "f32"),
    "QuantParams": lambda: H.QuantParams(cfg["rel_eps"] * (hi - lo), cfg["dims"], 32, "f32"),
    "compress": lambda: H.compress(raw, p),
    "negate": lambda: H.negate(s),
    "scalar_add": lambda: H.scalar_add(s, 3.5),
    "scalar_mul": lambda: H.scalar_mul(s, -1.25),
    "moments launch": lambda: O.moments_device(z, True),
    "mean(sync)": lambda: H.mean(z),
    "decompress": lambda: H.decompress(z),
}
for name, fn in fns.items():
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(30):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
        torch.cuda.synchronize()
    ts.sort()
    print(f"{name:24s} host {1e6 * ts[len(ts) // 2]:8.1f} us (median)")
