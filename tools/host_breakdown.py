"""Host cost of the pieces of one public-API call (median of 300 calls, no
synchronisation inside the loop): where the Python layer's launch latency
goes.

    python tools/host_breakdown.py
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2408_11971_b200 as H  # noqa: E402
from paper_2408_11971_b200 import device as D  # noqa: E402
from paper_2408_11971_b200 import ops as O  # noqa: E402
from paper_2408_11971_b200 import workloads as W  # noqa: E402

cfg = W.CONFIGS[2]
x = torch.from_numpy(W.config2()).cuda()
raw = H.RawArray(x, cfg["dims"], "f32")
lo, hi = raw.value_range()
p = H.QuantParams(cfg["rel_eps"] * (hi - lo), cfg["dims"], 32, "f32")
s = H.compress(raw, p)
torch.cuda.synchronize()
ctx = s.ctx
lib = ctx.lib
B = p.block_count
outl = ctx.empty(B, torch.int32)
po, pi = D.ptr(outl), D.ptr(s.outliers)


def t_of(fn, reps=300):
    for _ in range(20):
        fn()
    torch.cuda.synchronize()
    ts = []
    for i in range(reps):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
        if i % 50 == 49:
            torch.cuda.synchronize()
    ts.sort()
    return 1e6 * ts[len(ts) // 2]


rows = {
    "torch.empty(B,int32,cuda)": lambda: torch.empty(B, dtype=torch.int32, device="cuda"),
    "ctx.empty(B,int32)": lambda: ctx.empty(B, torch.int32),
    "tensor.data_ptr()": lambda: outl.data_ptr(),
    "device.ptr(tensor)": lambda: D.ptr(outl),
    "ctypes hsz_version()": lambda: lib.hsz_version(),
    "ctypes hsz_tile_count(n,k)": lambda: lib.hsz_tile_count(p.element_count, 32),
    "hsz_scalar_add C call (launch)": lambda: lib.hsz_scalar_add(pi, po, B, 7, ctx.err_ptr, ctx.handle),
    "torch.cuda.current_stream()": lambda: torch.cuda.current_stream(),
    "device.context()": lambda: D.context(),
    "ScalarBin.of": lambda: O.ScalarBin.of(3.5, p.eps),
    "DeviceStream(...)": lambda: D.DeviceStream(p, s.widths, outl, s.signs, s.payload, s.toff, ctx,
                                                 s.sign_cap, s.payload_cap),
    "H.scalar_add": lambda: H.scalar_add(s, 3.5),
    "H.negate": lambda: H.negate(s),
    "torch.zeros_like small add (torch launch)": lambda: outl.add_(0),
}
for name, fn in rows.items():
    print(f"{name:42s} {t_of(fn):8.2f} us")
