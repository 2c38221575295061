"""Generate golden fixtures by running the REFERENCE implementation itself.

Run in the build container (where ``/root/reference`` exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports the unmodified reference package from ``$HOSZP_REF_PATH`` (default
``/root/reference/pkg/src``), drives its public API on seeded inputs and
writes ``tests/golden/golden_streams.npz``.  The fixtures travel with the repo;
nothing at test time reads ``/root/reference``.

Each case records the inputs (bins or raw values + params), the reference's
serialized stream, its decoded bins and values, the bytes of every
homomorphically transformed stream, and mean / variance as exact float hex.
Error cases record the reference's exception class name.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = os.environ.get("HOSZP_REF_PATH", "/root/reference/pkg/src")
sys.path.insert(0, REF)
sys.dont_write_bytecode = True

import hoszp  # noqa: E402  (the reference)
from hoszp import ops  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden_streams.npz")


def _bytes(b: bytes) -> np.ndarray:
    return np.frombuffer(bytes(b), dtype=np.uint8).copy()


def _try(fn):
    try:
        return fn(), ""
    except Exception as exc:  # record the reference's exception class
        return None, type(exc).__name__


class Recorder:
    def __init__(self):
        self.arrays = {}
        self.n = 0

    def add(self, **kw):
        i = self.n
        self.n += 1
        for key, val in kw.items():
            self.arrays[f"c{i}_{key}"] = val
        return i


def params_arr(p):
    return np.array([p.eps], dtype=np.float64), np.array(p.dims, dtype=np.int64), \
        np.array([p.block_len], dtype=np.int64), np.array([0 if p.dtype == "f32" else 1])


def record_stream_case(rec, kind, p, src, stream_fn, scal_add, scal_mul):
    eps, dims, bl, dt = params_arr(p)
    s, err = _try(stream_fn)
    entry = dict(kind=np.array([kind]), eps=eps, dims=dims, block_len=bl, dtype=dt,
                 src=src, err=np.array([err]), sadd_s=np.array([scal_add]),
                 smul_s=np.array([scal_mul]))
    if s is None:
        rec.add(**entry)
        return
    entry["stream"] = _bytes(hoszp.serialize(s))
    q = hoszp.decode_to_quant(s)
    entry["bins_out"] = q.bins.copy()
    entry["values"] = hoszp.decompress(s).values.copy()
    for name, fn in (("neg", lambda: ops.negate(s)),
                     ("sadd", lambda: ops.scalar_add(s, scal_add)),
                     ("smul", lambda: ops.scalar_mul(s, scal_mul))):
        z, zerr = _try(fn)
        entry[f"{name}_err"] = np.array([zerr])
        if z is not None:
            entry[name] = _bytes(hoszp.serialize(z))
    m, merr = _try(lambda: ops.mean(s))
    v, verr = _try(lambda: ops.variance(s))
    entry["mean_hex"] = np.array([m.hex() if m is not None else merr])
    entry["var_hex"] = np.array([v.hex() if v is not None else verr])
    rec.add(**entry)


def random_params(rng, max_dim=40, dtypes=("f32", "f64"),
                  blocks=(1, 3, 4, 8, 32, 33, 128), eps_choices=(1e-1, 1e-2, 1e-3, 0.25)):
    nd = int(rng.integers(1, 4))
    dims = tuple(int(d) for d in rng.integers(1, max_dim, nd))
    return hoszp.QuantParams(float(rng.choice(eps_choices)), dims,
                             int(rng.choice(blocks)), str(rng.choice(dtypes)))


def random_bins(rng, p, hi):
    n = p.element_count
    b = rng.integers(-hi, hi, n)
    lo32, hi32 = max(-(2 ** 31), -hi), min(2 ** 31 - 1, hi)
    b[::p.block_len] = rng.integers(lo32, hi32, b[::p.block_len].size)
    return b


def main():
    rng = np.random.default_rng(20240822)
    rec = Recorder()

    # 1. the FORMAT.md worked example, compressed from raw values
    p = hoszp.QuantParams(0.01, (2, 2), 32, "f32")
    vals = np.array([-0.025, -0.025, -0.051, -0.052], dtype=np.float32)
    record_stream_case(rec, "raw", p, vals.astype(np.float64),
                       lambda: hoszp.compress(hoszp.RawArray(vals, (2, 2), "f32"), p),
                       0.67, 3.14)

    # 2. random bin streams through encode_from_quant (conftest.py:52-55 style)
    for hi, count in ((2 ** 12, 30), (2 ** 15, 30), (2 ** 20, 30), (2 ** 31, 12)):
        for _ in range(count):
            p = random_params(rng, max_dim=24)
            bins = random_bins(rng, p, hi)
            record_stream_case(rec, "bins", p, bins.astype(np.int64),
                               lambda: hoszp.encode_from_quant(hoszp.QuantArray(bins, p)),
                               float(rng.uniform(-50, 50)), float(rng.uniform(-20, 20)))

    # 3. raw fields through compress (uniform, smooth, masked with constants)
    for _ in range(40):
        p = random_params(rng, max_dim=32, eps_choices=(1e-1, 1e-2, 1e-3, 1e-4, 0.25))
        n = p.element_count
        kind = int(rng.integers(0, 3))
        if kind == 0:
            x = rng.uniform(-5, 5, n)
        elif kind == 1:
            t = np.linspace(0, 6 * np.pi, n)
            x = 3 * np.sin(t) + 0.5 * np.cos(7 * t)
        else:
            x = rng.normal(0, 1, n)
            x[: n // 2] = 1.0
        x = x.astype(p.numpy_dtype)
        record_stream_case(rec, "raw", p, x.astype(np.float64),
                           lambda: hoszp.compress(hoszp.RawArray(x, p.dims, p.dtype), p),
                           float(rng.uniform(-30, 30)), float(rng.uniform(-10, 10)))

    # 4. 32-element blocks at realistic sizes (the B200 fast path), f32
    for n, eps in ((4096 + 17, 1e-3), (8192, 1e-4), (32768 + 5, 0.0175), (50_000, 2e-5)):
        i = np.arange(n)
        x = (np.sin(2 * np.pi * 3 * i / n) * 50 + 280 + rng.normal(0, 0.5, n)).astype(np.float32)
        p = hoszp.QuantParams(eps, (n,), 32, "f32")
        record_stream_case(rec, "raw", p, x.astype(np.float64),
                           lambda: hoszp.compress(hoszp.RawArray(x, (n,), "f32"), p),
                           float(rng.uniform(-30, 30)), float(rng.uniform(-3, 3)))

    # 5. wide / near-63-bit bins (width 64 and the exact slow paths)
    for bins, k in (([-2, 2 ** 63 - 1], 2),
                    ([3, 2 ** 63 - 1, -(2 ** 63 - 1), 2 ** 62, -7, 0, 5, -(2 ** 62), 11], 4),
                    ([0, 2 ** 62, -(2 ** 62), 5], 4),
                    ([5] * 40 + [2 ** 40, -(2 ** 40)] * 12, 32),
                    ([2 ** 31 - 1] + [2 ** 62] * 31 + [-(2 ** 31)] * 32, 32)):
        bins = np.array(bins, dtype=np.int64)
        p = hoszp.QuantParams(0.1, (bins.size,), k, "f64")
        record_stream_case(rec, "bins", p, bins,
                           lambda: hoszp.encode_from_quant(hoszp.QuantArray(bins, p)),
                           1.0, 0.25)

    # 6. constant blocks, all-zero and tail blocks with block_len 32
    for bins in (np.zeros(70, np.int64), np.full(64, 7, np.int64),
                 np.repeat(np.arange(-5, 6), 32)[:345],
                 np.concatenate([np.full(32, -3), np.arange(32), np.full(5, 9)])):
        p = hoszp.QuantParams(0.01, (bins.size,), 32, "f32")
        record_stream_case(rec, "bins", p, bins.astype(np.int64),
                           lambda: hoszp.encode_from_quant(hoszp.QuantArray(bins, p)),
                           0.67, 3.14)

    # 7. error cases
    for vals, eps, dt in (([1e80], 1e-300, "f64"), ([1.0e12 + 0.5], 1e-7, "f64")):
        p = hoszp.QuantParams(eps, (1,), 32, dt)
        v = np.array(vals, dtype=np.float64)
        record_stream_case(rec, "raw", p, v,
                           lambda: hoszp.compress(hoszp.RawArray(v, (1,), dt), p), 1.0, 1.0)
    for bins, eps, sa in (([-(2 ** 31), 0, 0], 0.01, 0.0), ([2 ** 31 - 1, 0, 0], 0.5, 100.0)):
        bins = np.array(bins, dtype=np.int64)
        p = hoszp.QuantParams(eps, (3,), 32, "f32")
        record_stream_case(rec, "bins", p, bins,
                           lambda: hoszp.encode_from_quant(hoszp.QuantArray(bins, p)),
                           sa, 1e6)

    # 8. boundary inputs sitting exactly on bin edges (the repair pass)
    for eps in (0.01, 0.0175, 0.1, 2.0 ** -7):
        m = np.arange(-300, 300)
        x = ((2 * m - 1) * eps).astype(np.float64)
        p = hoszp.QuantParams(eps, (x.size,), 32, "f64")
        record_stream_case(rec, "raw", p, x,
                           lambda: hoszp.compress(hoszp.RawArray(x, (x.size,), "f64"), p),
                           3.5, -1.25)
        xf = x.astype(np.float32)
        pf = hoszp.QuantParams(eps, (x.size,), 32, "f32")
        record_stream_case(rec, "raw", pf, xf.astype(np.float64),
                           lambda: hoszp.compress(hoszp.RawArray(xf, (x.size,), "f32"), pf),
                           3.5, -1.25)

    rec.arrays["count"] = np.array([rec.n])
    np.savez_compressed(OUT, **rec.arrays)
    print(f"wrote {rec.n} cases to {OUT} ({os.path.getsize(OUT)} bytes)")


if __name__ == "__main__":
    main()
