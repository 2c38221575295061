"""Adversarial streams at the edges of the register (fast) paths, every op
against the oracle: same-sign residual ramps at the widths around each fast
path's width bound (16/17, 22-27), outliers straddling the |o| < 2^29 fast
bound, bins around 2^30 (the smul / element-wise int32 bounds) and 2^31.
Results must match byte for byte (streams), bit for bit (floats), and raise
the same error class."""

import numpy as np
import pytest

import hoszp_oracle as O

pytestmark = pytest.mark.gpu
EPS = 0.01
N = 4096 * 3 + 45


@pytest.fixture(scope="module")
def H():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2408_11971_b200 as mod

    return mod


def _ramps(rng, w, o_lo, o_hi):
    blk = np.arange(N) // 32
    d = rng.integers(1 << (w - 1), 1 << w, N).astype(np.int64)
    d *= rng.choice([-1, 1], blk[-1] + 1)[blk]
    d[::32] = rng.integers(o_lo, o_hi, d[::32].size)
    bins = np.zeros(N, dtype=np.int64)
    for b in range(blk[-1] + 1):
        sl = slice(32 * b, min(32 * b + 32, N))
        bins[sl] = np.cumsum(d[sl])
    return bins


def _bins(kind, seed):
    rng = np.random.default_rng(seed)
    if kind.startswith("ramp"):
        return _ramps(rng, int(kind[4:]), -(1 << 20), 1 << 20)
    if kind == "edge_outliers":
        # block starts at +-(2^29 - 1), +-2^29, +-(2^29 + 1); small residuals
        bins = rng.integers(-300, 300, N).astype(np.int64)
        opts = np.array([(1 << 29) - 1, 1 << 29, (1 << 29) + 1])
        starts = rng.choice(opts, bins[::32].size) * rng.choice([-1, 1], bins[::32].size)
        bins += np.repeat(starts, 32)[:N]
        return bins
    if kind == "near_2p30":
        base = rng.choice([(1 << 30) - 64, -(1 << 30) + 64], N // 32 + 1)
        return np.repeat(base, 32)[:N] + rng.integers(-63, 63, N)
    if kind == "near_2p31":
        base = rng.choice([(1 << 31) - 2000, -(1 << 31) + 2000], N // 32 + 1)
        return (np.repeat(base, 32)[:N] + rng.integers(-1000, 1000, N)).astype(np.int64)
    raise ValueError(kind)


KINDS = ["ramp16", "ramp17", "ramp22", "ramp23", "ramp24", "ramp25", "ramp26", "ramp27",
         "edge_outliers", "near_2p30", "near_2p31"]


def _pair(H, kind, seed):
    bins = _bins(kind, seed)
    try:
        ref = O.encode_bins(bins, EPS, (N,), 32, "f32")
    except O.OracleError:
        pytest.skip("bins not encodable (outlier beyond int32)")
    s = H.deserialize(O.serialize(ref))
    return s, ref


def _run(fn):
    try:
        return fn()
    except Exception as e:          # the class is the result
        return type(e).__name__


def _same(got, want):
    if isinstance(want, dict):
        want = O.serialize(want)
    if isinstance(got, str) or isinstance(want, str):
        assert got == want
    elif isinstance(want, bytes):
        assert got == want
    elif isinstance(want, np.ndarray):
        assert np.asarray(got).tobytes() == want.tobytes()
    else:
        assert got == want


@pytest.mark.parametrize("kind", KINDS)
def test_unary_ops_at_fast_path_edges(H, kind):
    s, ref = _pair(H, kind, 1)
    # decode paths
    _same(_run(lambda: np.asarray(H.decode_to_quant(s).bins)), O.decode_bins(ref))
    _same(_run(lambda: H.decompress(s).values), O.decompress(ref))
    _same(_run(lambda: H.decompress(s, out_dtype=np.float64).values), O.decompress(ref, True))
    S, Q = O.moments(ref)
    _same(_run(lambda: H.mean(s)), O.mean_from(S, N, EPS))
    _same(_run(lambda: H.variance(s)), O.variance_from(S, Q, N, EPS))
    _same(_run(lambda: H.block_means(s)), O.block_means(ref))
    # stream ops
    _same(_run(lambda: H.serialize(H.negate(s))), _run(lambda: O.serialize(O.negate(ref))))
    for v in (3.5, -1e6):
        _same(_run(lambda: H.serialize(H.scalar_add(s, v))),
              _run(lambda: O.serialize(O.scalar_add(ref, v))))
    for v in (-1.25, 0.75, 3.0, 1e4, -3.7e6):
        _same(_run(lambda: H.serialize(H.scalar_mul(s, v))),
              _run(lambda: O.serialize(O.scalar_mul(ref, v))))


@pytest.mark.parametrize("ka,kb", [("ramp24", "ramp24"), ("ramp22", "edge_outliers"),
                                   ("near_2p30", "near_2p30"), ("ramp26", "near_2p30"),
                                   ("edge_outliers", "edge_outliers"), ("ramp17", "ramp25"),
                                   ("near_2p31", "ramp16")])
def test_binary_ops_at_fast_path_edges(H, ka, kb):
    a, ra = _pair(H, ka, 2)
    b, rb = _pair(H, kb, 3)
    _same(_run(lambda: H.serialize(H.elementwise_add(a, b))),
          _run(lambda: O.serialize(O.elementwise_add(ra, rb))))
    _same(_run(lambda: H.serialize(H.elementwise_sub(a, b))),
          _run(lambda: O.serialize(O.elementwise_sub(ra, rb))))
    _same(_run(lambda: H.serialize(H.hadamard(a, b))),
          _run(lambda: O.serialize(O.hadamard(ra, rb))))
    _same(_run(lambda: H.covariance(a, b)), _run(lambda: O.covariance(ra, rb)))
    _same(_run(lambda: H.ssim_global(a, b)), _run(lambda: O.ssim_global(ra, rb)))
    from paper_2408_11971_b200 import distsim

    _same(_run(lambda: H.serialize(distsim.aggregate_homomorphic([a, b, a]))),
          _run(lambda: O.serialize(O.aggregate_homomorphic([ra, rb, ra]))))


def _ramps_k(rng, w, k, n):
    blk = np.arange(n) // k
    d = rng.integers(1 << (w - 1), 1 << w, n).astype(np.int64)
    d *= rng.choice([-1, 1], blk[-1] + 1)[blk]
    d[::k] = rng.integers(-(1 << 28), 1 << 28, d[::k].size)
    bins = np.zeros(n, dtype=np.int64)
    for b in range(blk[-1] + 1):
        sl = slice(k * b, min(k * b + k, n))
        bins[sl] = np.cumsum(d[sl])
    return bins


@pytest.mark.parametrize("k", [8, 33, 128])
@pytest.mark.parametrize("w", [20, 24, 26, 27])
def test_generic_block_length_ramps(H, k, w):
    """The generic (k != 32) decoder's register path is bounded at width 26;
    ramps of 127 same-sign residuals at those widths leave int32."""
    n = 128 * k * 2 + 17
    rng = np.random.default_rng(k * 100 + w)
    bins = _ramps_k(rng, min(w, 30 if k <= 8 else w), k, n)
    try:
        ref = O.encode_bins(bins, EPS, (n,), k, "f32")
    except O.OracleError:
        pytest.skip("bins not encodable")
    s = H.deserialize(O.serialize(ref))
    _same(_run(lambda: np.asarray(H.decode_to_quant(s).bins)), O.decode_bins(ref))
    _same(_run(lambda: H.decompress(s, out_dtype=np.float64).values), O.decompress(ref, True))
    S, Q = O.moments(ref)
    _same(_run(lambda: H.mean(s)), O.mean_from(S, n, EPS))
    _same(_run(lambda: H.variance(s)), O.variance_from(S, Q, n, EPS))
    _same(_run(lambda: H.serialize(H.scalar_mul(s, -0.75))),
          _run(lambda: O.serialize(O.scalar_mul(ref, -0.75))))
    _same(_run(lambda: H.serialize(H.elementwise_add(s, s))),
          _run(lambda: O.serialize(O.elementwise_add(ref, ref))))


@pytest.mark.parametrize("case", ["saw22", "saw24", "saw26", "near_2p31", "near_2p29_starts",
                                  "huge_small_eps", "mixed_magnitudes"])
def test_compress_at_fast_path_edges(H, case):
    """compress (quantize + encode in one pass) on inputs whose bins sit at
    the encoder's register-path bounds; stream bytes or error class."""
    import zlib

    rng = np.random.default_rng(zlib.crc32(case.encode()))
    n = 4096 * 3 + 45
    eps = 0.01
    i = np.arange(n)
    if case.startswith("saw"):
        step = 2 * eps * (1 << (int(case[3:]) - 1)) * 1.3
        x = (i % 32) * step * rng.choice([-1, 1], n // 32 + 1)[i // 32]
    elif case == "near_2p31":
        x = 2 * eps * ((1 << 31) + rng.integers(-5000, 5000, n)) * rng.choice([-1, 1], n)
        x[::32] = rng.normal(0, 100, x[::32].size)           # outliers fit; residuals ~2^32
    elif case == "near_2p29_starts":
        x = 2 * eps * ((1 << 29) + rng.integers(-40, 40, n)) * rng.choice([-1, 1], n // 32 + 1)[i // 32]
    elif case == "huge_small_eps":
        x = rng.normal(0, 1e30, n)
        eps = 1e-10
    else:
        x = rng.normal(0, 1, n) * 10.0 ** rng.integers(-3, 7, n)
    x = x.astype(np.float32)
    got = _run(lambda: H.serialize(H.compress(H.RawArray(x, (n,), "f32"),
                                              H.QuantParams(eps, (n,), 32, "f32"))))
    want = _run(lambda: O.serialize(O.compress(x, eps, (n,), 32, "f32")))
    _same(got, want)
