"""PCIe bandwidth on the bench box: pinned H2D alone, D2H alone, and both
directions at once (what the pipelined e2e leg overlaps)."""
import json
import time

import torch

h_in = torch.empty(100_000_000, dtype=torch.uint8, pin_memory=True)
h_out = torch.empty(135_000_000, dtype=torch.uint8, pin_memory=True)
d_in = torch.empty(h_in.numel(), dtype=torch.uint8, device="cuda")
d_out = torch.empty(h_out.numel(), dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=10):
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    return min(ts)


def h2d():
    with torch.cuda.stream(s1):
        d_in.copy_(h_in, non_blocking=True)


def d2h():
    with torch.cuda.stream(s2):
        h_out.copy_(d_out, non_blocking=True)


def both():
    h2d()
    d2h()


t1, t2, t3 = timed(h2d), timed(d2h), timed(both)
print(json.dumps({"h2d_GBps": round(1e-9 * h_in.numel() / t1, 1),
                  "d2h_GBps": round(1e-9 * h_out.numel() / t2, 1),
                  "both_ms": round(1e3 * t3, 3),
                  "both_GBps_combined": round(1e-9 * (h_in.numel() + h_out.numel()) / t3, 1),
                  "serial_ms": round(1e3 * (t1 + t2), 3)}))
