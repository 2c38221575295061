"""Randomised stress of the shipped kernels in ONE process (workspace, ticket
and epoch state carried across hundreds of launches of every kind), checked
against the CPU oracle.  A watchdog dumps the Python stacks and exits if any
single iteration takes longer than 60 s (a hung kernel).

    python tools/stress.py [iterations] [seed]
"""
import faulthandler
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import hoszp_oracle as O  # noqa: E402
import paper_2408_11971_b200 as H  # noqa: E402
from paper_2408_11971_b200 import distsim  # noqa: E402


def field(rng, n):
    kind = int(rng.integers(0, 4))
    i = np.arange(n)
    if kind == 0:
        x = np.sin(i / rng.uniform(20, 2000)) * rng.uniform(1, 100)
    elif kind == 1:
        x = rng.normal(0, rng.uniform(0.1, 10), n)
        x[(i // 4096) % 3 == 0] = 1.5
    elif kind == 2:
        x = np.exp(rng.normal(0, 1.5, n))
    else:
        x = np.cumsum(rng.normal(0, 1, n))
    return x.astype(np.float32)


def run(iters=200, seed=0, verbose=True):
    rng = np.random.default_rng(seed)
    t_start = time.time()
    for it in range(iters):
        faulthandler.dump_traceback_later(60, exit=True)
        n = int(rng.integers(1, 200_000)) if rng.random() < 0.7 else int(rng.integers(200_000, 3_000_000))
        k = 32 if rng.random() < 0.85 else int(rng.choice((1, 8, 33, 128)))
        xa, xb = field(rng, n), field(rng, n)
        rel = float(rng.choice((1e-2, 1e-3, 1e-4, 1e-5)))
        span = float(max(xa.max(), xb.max()) - min(xa.min(), xb.min())) or 1.0
        p = H.QuantParams(rel * span, (n,), k, "f32")
        ra = H.RawArray(torch.from_numpy(xa).cuda(), (n,), "f32")
        rb = H.RawArray(torch.from_numpy(xb).cuda(), (n,), "f32")
        a, b = H.compress(ra, p), H.compress(rb, p)
        op = int(rng.integers(0, 8))
        s_add, s_mul = float(rng.uniform(-50, 50)), float(rng.uniform(-3, 3))
        try:
            if op == 0:
                z = H.scalar_mul(H.scalar_add(H.negate(a), s_add), s_mul)
            elif op == 1:
                z = H.elementwise_add(a, b)
            elif op == 2:
                z = H.elementwise_sub(a, b)
            elif op == 3:
                z = H.hadamard(a, b)
            elif op == 4:
                z = distsim.aggregate_homomorphic([a, b, a])
            elif op == 5:
                z = H.encode_from_quant(H.decode_to_quant(a))
            else:
                z = a
            got = H.serialize(z.to_host())
            m, v = H.mean(z), H.variance(z)
            vals = H.decompress(z).values.cpu().numpy()
        except H.HoszpError as e:          # overflow classes are legitimate outcomes
            got, m, v, vals = type(e).__name__, None, None, None
        if n <= 200_000:                   # the oracle checks the small cases
            oa = O.compress(xa, p.eps, (n,), k, "f32")
            ob = O.compress(xb, p.eps, (n,), k, "f32")
            try:
                if op == 0:
                    want = O.scalar_mul(O.scalar_add(O.negate(oa), s_add), s_mul)
                elif op == 1:
                    want = O.elementwise_add(oa, ob)
                elif op == 2:
                    want = O.elementwise_sub(oa, ob)
                elif op == 3:
                    want = O.hadamard(oa, ob)
                elif op == 4:
                    want = O.aggregate_homomorphic([oa, ob, oa])
                else:
                    want = oa
                if want is not None:
                    ws = O.serialize(want)
                    assert got == ws, f"iter {it}: op {op} n {n} k {k} stream mismatch"
                    if m is not None:
                        S, Q = O.moments(want)
                        assert m == O.mean_from(S, n, p.eps) and v == O.variance_from(S, Q, n, p.eps)
                        assert vals.tobytes() == O.decompress(want).tobytes()
            except O.OracleError as e:
                assert isinstance(got, str), f"iter {it}: oracle raised {type(e).__name__}, GPU did not"
        faulthandler.cancel_dump_traceback_later()
        if verbose and it % 25 == 0:
            print(f"iter {it} n={n} k={k} op={op} ok  ({time.time() - t_start:.1f}s)", flush=True)
    if verbose:
        print(f"stress ok: {iters} iterations in {time.time() - t_start:.1f}s")


if __name__ == "__main__":
    run(int(sys.argv[1]) if len(sys.argv) > 1 else 200, int(sys.argv[2]) if len(sys.argv) > 2 else 0)
