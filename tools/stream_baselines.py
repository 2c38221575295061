"""Streaming baselines at the bench sizes: torch's own elementwise/reduction
kernels next to ours, timed the same way as tools/time_ops.py (L2 read-flush,
spin pre-roll, mean of reps).  Tells fixed launch/ramp cost from kernel
design for the small streaming ops."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2408_11971_b200 as H  # noqa: E402
from paper_2408_11971_b200 import workloads as W  # noqa: E402


def t_of(fn, flush, reps=20):
    ts = []
    for _ in range(reps + 2):
        flush.view(torch.int64).max()
        torch.cuda._sleep(400_000)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return round(1e3 * statistics.mean(ts[2:]), 2)


flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
out = {}
for cfg in (2, 4):
    c = W.CONFIGS[cfg]
    x = W.field(cfg, device="cuda")
    x = (x if torch.is_tensor(x) else torch.from_numpy(x)).cuda().reshape(-1).contiguous()
    raw = H.RawArray(x, c["dims"], "f32")
    lo, hi = raw.value_range()
    p = H.QuantParams(c["rel_eps"] * (hi - lo), c["dims"], 32, "f32")
    s = H.compress(raw, p)
    o = s.outliers
    o2 = torch.empty_like(o)
    y = torch.empty_like(x)
    r = {
        "torch_aminmax_field": t_of(lambda: torch.aminmax(x), flush),
        "torch_copy_field": t_of(lambda: y.copy_(x), flush),
        "torch_add_outliers": t_of(lambda: torch.add(o, 7, out=o2), flush),
        "torch_copy_outliers": t_of(lambda: o2.copy_(o), flush),
        "hsz_scalar_add": t_of(lambda: H.scalar_add(s, c["sadd"]), flush),
        "hsz_negate": t_of(lambda: H.negate(s), flush),
        "field_MB": x.numel() * 4 / 1e6, "outliers_MB": o.numel() * 4 / 1e6,
    }
    out[f"config{cfg}"] = r
print(json.dumps(out, indent=1))
