"""Encoder-interleaving stress: every persistent look-back encoder (compress,
scalar_mul, elementwise add/sub, hadamard's re-encode, encode_from_quant) and
the tile-offset rebuild, launched back to back in ONE process on random sizes
(so the persistent grids vary from 1 CTA to the whole GPU) with the workspace
ticket / epoch state carried across every launch.

Each iteration runs its encoders twice and requires identical bytes (a
deadlock, a lost tile or a mis-placed tile would break that); every
`--oracle-every`-th iteration is also checked against the CPU oracle.  The
look-back watchdog is armed (hsz_set_lookback_watchdog), so a protocol
failure raises DeviceTimeout instead of hanging; a Python-side watchdog
dumps the stacks if one iteration takes longer than 60 s.

    python tools/stress_encoders.py [iterations] [seed] [--oracle-every K]
"""
import argparse
import faulthandler
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2408_11971_b200 as H  # noqa: E402


def _field(rng, n):
    kind = int(rng.integers(0, 4))
    if kind == 0:
        x = np.cumsum(rng.normal(0, rng.uniform(0.1, 3), n))
    elif kind == 1:
        x = np.exp(rng.normal(0, 1.5, n))
    elif kind == 2:
        x = np.sin(np.arange(n) / rng.uniform(10, 500)) * rng.uniform(1, 50)
    else:
        # tiles alternating between quiet and very noisy data: packed tile
        # sizes jump between a few hundred bytes and most of the staging ring
        # (the pattern behind the round-2 ring deadlock)
        amp = np.where((np.arange(n) // 4096) % 2 == 0, 1e-3, 1.0) * rng.uniform(0.5, 2)
        x = rng.normal(0, 1, n) * amp
    return torch.from_numpy(x.astype(np.float32)).cuda()


def _bytes(ds):
    sb, pb = ds.totals()
    return (ds.widths, ds.outliers, ds.signs[:sb], ds.payload[:pb])


def _same(a, b):
    return all(x.numel() == y.numel() and torch.equal(x, y) for x, y in zip(_bytes(a), _bytes(b)))


def run(iters=2000, seed=0, oracle_every=50, verbose=True):
    import hoszp_oracle as O
    from paper_2408_11971_b200 import _native

    lib = _native.load()
    old = lib.hsz_set_lookback_watchdog(1 << 20)     # well above any legitimate wait
    rng = np.random.default_rng(seed)
    launches = 0
    t0 = time.time()
    try:
        for it in range(iters):
            faulthandler.dump_traceback_later(60, exit=True)
            r = rng.random()
            n = int(rng.integers(1, 5_000)) if r < 0.3 else (
                int(rng.integers(5_000, 400_000)) if r < 0.9 else int(rng.integers(400_000, 4_000_000)))
            xa, xb = _field(rng, n), _field(rng, n)
            span = float(torch.maximum(xa.max(), xb.max()) - torch.minimum(xa.min(), xb.min())) or 1.0
            eps = float(rng.choice((1e-2, 1e-3, 1e-4))) * span
            p = H.QuantParams(eps, (n,), 32, "f32")
            ra, rb = H.RawArray(xa, (n,), "f32"), H.RawArray(xb, (n,), "f32")
            sm = float(rng.choice((-1.25, 3.0, 0.5, -7.0))) * eps * 2
            ops = [
                ("compress_a", lambda: H.compress(ra, p)),
                ("compress_b", lambda: H.compress(rb, p)),
            ]
            a = ops[0][1]()
            b = ops[1][1]()
            ops += [
                ("scalar_mul", lambda: H.scalar_mul(a, sm)),
                ("eadd", lambda: H.elementwise_add(a, b)),
                ("esub", lambda: H.elementwise_sub(a, b)),
                ("hadamard", lambda: H.hadamard(a, b)),
                ("encode_from_quant", lambda: H.encode_from_quant(H.decode_to_quant(a))),
                ("from_sections", lambda: H.DeviceStream.from_sections(
                    p, a.widths, a.outliers.view(torch.uint8), *_bytes(a)[2:])),
            ]
            order = rng.permutation(len(ops))
            first, second = {}, {}
            for i in order:                     # interleaved in a random order, twice
                name, fn = ops[i]
                try:
                    first[name] = fn()
                except H.HoszpError as e:
                    first[name] = type(e).__name__
                launches += 1
            for i in rng.permutation(len(ops)):
                name, fn = ops[i]
                try:
                    second[name] = fn()
                except H.HoszpError as e:
                    second[name] = type(e).__name__
                launches += 1
            for name in first:
                u, v = first[name], second[name]
                if isinstance(u, str) or isinstance(v, str):
                    assert u == v if isinstance(u, str) and isinstance(v, str) else False, \
                        f"iter {it} {name}: {u!r} vs {v!r}"
                    continue
                assert _same(u, v), f"iter {it} {name}: two launches gave different bytes (n={n})"
                u.check()
            if oracle_every and it % oracle_every == 0 and n <= 400_000:
                oa = O.compress(xa.cpu().numpy(), eps, (n,), 32, "f32")
                ob = O.compress(xb.cpu().numpy(), eps, (n,), 32, "f32")
                want = {"compress_a": oa, "compress_b": ob, "eadd": O.elementwise_add(oa, ob),
                        "esub": O.elementwise_sub(oa, ob)}
                for name, w in want.items():
                    if not isinstance(first[name], str):
                        assert H.serialize(first[name].to_host()) == O.serialize(w), \
                            f"iter {it} {name}: differs from the oracle"
            faulthandler.cancel_dump_traceback_later()
            if verbose and it % 250 == 0:
                print(f"iter {it} n={n} launches={launches} ({time.time() - t0:.1f}s)", flush=True)
    finally:
        lib.hsz_set_lookback_watchdog(old)
    if verbose:
        print(f"stress_encoders ok: {iters} iterations, {launches} encoder launches in "
              f"{time.time() - t0:.1f}s")
    return launches


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("iters", type=int, nargs="?", default=2000)
    ap.add_argument("seed", type=int, nargs="?", default=0)
    ap.add_argument("--oracle-every", type=int, default=50)
    a = ap.parse_args()
    run(a.iters, a.seed, a.oracle_every)
