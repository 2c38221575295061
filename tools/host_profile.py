"""cProfile of the public-API host path (no synchronisation inside the loop):
which Python frames the launch latency of each op is spent in.

    python tools/host_profile.py [op]
"""
import cProfile
import os
import pstats
import sys

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
ops = {
    "compress": lambda: H.compress(raw, p),
    "scalar_mul": lambda: H.scalar_mul(s, -1.25),
    "negate": lambda: H.negate(s),
    "mean": lambda: H.mean(z),
    "decompress": lambda: H.decompress(z),
    "value_range": lambda: H.RawArray(x, cfg["dims"], "f32").value_range(),
}
for name in (sys.argv[1:] or list(ops)):
    fn = ops[name]
    for _ in range(20):
        fn()
    torch.cuda.synchronize()
    pr = cProfile.Profile()
    pr.enable()
    for i in range(200):
        fn()
        if i % 20 == 19:
            torch.cuda.synchronize()
    pr.disable()
    torch.cuda.synchronize()
    print(f"===== {name} (200 calls)")
    pstats.Stats(pr).sort_stats("tottime").print_stats(14)
