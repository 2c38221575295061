"""Run each hot-path op a few times on a config field (for ncu / nsys-less profiling).

    python tools/prof_ops.py [--config 2] [--reps 3]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2408_11971_b200 as H  # noqa: E402
from paper_2408_11971_b200 import ops as O  # noqa: E402
from paper_2408_11971_b200 import workloads as W  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
cfg = W.CONFIGS[a.config]
x = torch.from_numpy(W.field(a.config)).cuda().contiguous()   # the bench's host field
raw = H.RawArray(x, cfg["dims"], "f32")
lo, hi = raw.value_range()
p = H.QuantParams(cfg["rel_eps"] * (hi - lo), cfg["dims"], 32, "f32")
for _ in range(a.reps):
    s = H.compress(raw, p)
    z = H.negate(s)
    z = H.scalar_add(z, cfg["sadd"])
    z = H.scalar_mul(z, cfg["smul"])
    O.moments_device(z, False)
    O.moments_device(z, True)
    H.decompress(z)
torch.cuda.synchronize()
s.check()
print("ok", p.eps, s.serialized_size)
