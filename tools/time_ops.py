"""Device time of each hot-path op launched alone (L2 flushed first).

A ~0.3 ms spin kernel is queued after the flush so the host enqueues the op
while the GPU is busy: the CUDA-event interval then holds device time only,
not Python launch latency.

    python tools/time_ops.py [--config 2] [--reps 20] [--ops compress,decompress]
"""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2408_11971_b200 as H  # noqa: E402
from paper_2408_11971_b200 import ops as O  # noqa: E402
from paper_2408_11971_b200 import workloads as W  # noqa: E402


FLUSH = os.environ.get("HSZ_FLUSH", "read")


def do_flush(flush):
    """Evict L2 between timed launches.  "read" leaves clean lines (a write
    flush leaves ~126 MB of dirty lines whose write-back the next kernel pays)."""
    if FLUSH == "write":
        flush.fill_(1)
    elif FLUSH == "read":
        flush.view(torch.int64).max()


def device_times(fns, flush, reps):
    out = {}
    for name, fn in fns.items():
        ts = []
        for _ in range(reps + 2):
            if FLUSH != "none":
                do_flush(flush)
            torch.cuda._sleep(400_000)          # keep the GPU busy while the host enqueues
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        out[name] = statistics.mean(ts[2:])
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--ops", default="")
    a = ap.parse_args()
    cfg = W.CONFIGS[a.config]
    x = W.field(a.config)
    if not torch.is_tensor(x):
        x = torch.from_numpy(x)
    x = x.cuda().contiguous().reshape(-1)
    raw = H.RawArray(x, cfg["dims"], "f32")
    lo, hi = raw.value_range()
    p = H.QuantParams(cfg["rel_eps"] * (hi - lo), cfg["dims"], 32, "f32")
    if a.ops == "compress":        # (debug builds: the stream may be garbage)
        flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
        t = device_times({"compress": lambda: H.compress(raw, p)}, flush, a.reps)
        print(json.dumps({k: round(v * 1e3, 2) for k, v in t.items()}))
        return
    s = H.compress(raw, p)
    z0 = H.scalar_add(H.negate(s), cfg["sadd"])
    z = H.scalar_mul(z0, cfg["smul"])
    qz = H.decode_to_quant(z)
    ctx = s.ctx
    wsp, wsb = ctx.workspace(1, 1)
    mm = ctx.empty(2, torch.float64)
    from paper_2408_11971_b200 import _native as N
    from paper_2408_11971_b200.device import ptr
    fns = {
        "minmax": lambda: N.check(ctx.lib.hsz_minmax(ptr(x), N.HSZ_F32, x.numel(), ptr(mm), ctx.err_ptr,
                                                     wsp, wsb, ctx.handle), "hsz_minmax"),
        "compress": lambda: H.compress(raw, p),
        "negate": lambda: H.negate(s),
        "scalar_add": lambda: H.scalar_add(s, cfg["sadd"]),
        "scalar_mul": lambda: H.scalar_mul(z0, cfg["smul"]),
        "mean": lambda: O.moments_device(z, False),
        "variance": lambda: O.moments_device(z, True),
        "decompress": lambda: H.decompress(z),
        "elementwise_add": lambda: H.elementwise_add(s, z0),
        "decode_to_quant": lambda: H.decode_to_quant(z),
        "encode_from_quant": lambda: H.encode_from_quant(qz),
        "decompress_f64": lambda: H.decompress(z, out_dtype=np.float64),
    }
    if a.ops:
        fns = {k: v for k, v in fns.items() if k in a.ops.split(",")}
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    t = device_times(fns, flush, a.reps)
    z.check()
    print(json.dumps({k: round(v * 1e3, 2) for k, v in t.items()}))   # microseconds


if __name__ == "__main__":
    main()
