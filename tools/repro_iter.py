"""One iteration of tools/stress.py's sequence in isolation (the rng is replayed on
the CPU up to it).  python tools/repro_iter.py <seed> <iter> [sub-steps]"""
import os
import sys
import time
import faulthandler

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2408_11971_b200 as H  # noqa: E402
from paper_2408_11971_b200 import _native, distsim  # noqa: E402
import stress  # noqa: E402

lib = _native.load()
lib.hsz_set_lookback_watchdog(1 << 14)
lib.hsz_set_host_wait_timeout(15.0)
seed, target = int(sys.argv[1]), int(sys.argv[2])
mode = sys.argv[3] if len(sys.argv) > 3 else "op"
rng = np.random.default_rng(seed)
for it in range(target + 1):
    n = int(rng.integers(1, 200_000)) if rng.random() < 0.7 else int(rng.integers(200_000, 3_000_000))
    k = 32 if rng.random() < 0.85 else int(rng.choice((1, 8, 33, 128)))
    xa, xb = stress.field(rng, n), stress.field(rng, n)
    rel = float(rng.choice((1e-2, 1e-3, 1e-4, 1e-5)))
    op = int(rng.integers(0, 8))
    s_add, s_mul = float(rng.uniform(-50, 50)), float(rng.uniform(-3, 3))
faulthandler.dump_traceback_later(120, exit=True)
span = float(max(xa.max(), xb.max()) - min(xa.min(), xb.min())) or 1.0
p = H.QuantParams(rel * span, (n,), k, "f32")
print(f"iter {it} n={n} k={k} op={op} rel={rel} eps={p.eps} lib={os.environ.get('HSZ_B200_LIB','default')}", flush=True)
ra = H.RawArray(torch.from_numpy(xa).cuda(), (n,), "f32")
rb = H.RawArray(torch.from_numpy(xb).cuda(), (n,), "f32")
a, b = H.compress(ra, p), H.compress(rb, p)
a.check(); b.check()
print("compressed", flush=True)
try:
    if mode == "op":
        z = H.hadamard(a, b)
        z.check()
        print("hadamard ok", z.totals(), flush=True)
    else:
        qa = H.decode_to_quant(a); qb = H.decode_to_quant(b)
        torch.cuda.synchronize()
        prod = qa.bins.double() * qb.bins.double() * (2 * p.eps)
        bins = torch.where(prod < 0, -torch.floor(prod.abs() + 0.5), torch.floor(prod.abs() + 0.5)).to(torch.int64)
        print("bins absmax", int(bins.abs().max()), "tiles wide", int((bins.abs() >= 2**30).sum()), flush=True)
        z = H.encode_from_quant(H.QuantArray(bins, p))
        z.check()
        print("encode ok", z.totals(), flush=True)
except H.HoszpError as e:
    print("   ->", type(e).__name__, str(e)[:100], flush=True)
print("done")
