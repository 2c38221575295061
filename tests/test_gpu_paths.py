"""GPU parity of the less-travelled paths of the block_len-32 kernels, each
checked byte-exactly against the CPU oracle:

* compress: TMA tensor loads vs plain loads (misaligned input), the stream's
  partial last block on the TMA path, fields whose bins reach 2^30 (the exact
  warp-per-block tile path) next to ordinary tiles, elements inside the
  float32 certificate margin (exact float64 fallback per element);
* decode pipeline (decompress / mean / variance) and scalar_mul: tiles wider
  than the register decode (widths > 24), tiles whose payload exceeds the
  staging buffer (read in place), outliers beyond 2^29, scalars beyond 2^23
  and products beyond 2^30 (exact fallback), overflow error classes.
"""

import numpy as np
import pytest

import hoszp_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def H():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2408_11971_b200 as mod

    return mod


def _check_stream(H, s, ref):
    assert H.serialize(s) == O.serialize(ref)


def _full_check(H, x, eps, dims):
    p = H.QuantParams(eps, dims, 32, "f32")
    s = H.compress(H.RawArray(x, dims, "f32"), p)
    ref = O.compress(x, eps, dims, 32, "f32")
    _check_stream(H, s, ref)
    assert H.decompress(s).values.tobytes() == O.decompress(ref).tobytes()
    S, Q = O.moments(ref)
    assert H.mean(s) == O.mean_from(S, x.size, eps)
    assert H.variance(s) == O.variance_from(S, Q, x.size, eps)
    return s, ref


@pytest.mark.parametrize("n", [4096 * 3, 4096 * 3 + 7, 4096 * 40 + 31, 128 * 32 + 1, 5000])
def test_compress_tma_and_tail(H, n):
    rng = np.random.default_rng(n)
    x = np.cumsum(rng.normal(0, 0.3, n)).astype(np.float32)
    _full_check(H, x, 0.01, (n,))


def test_compress_misaligned_input_plain_loads(H):
    import torch

    n = 4096 * 8 + 5
    rng = np.random.default_rng(7)
    x = np.cumsum(rng.normal(0, 0.3, n + 1)).astype(np.float32)
    xd = torch.from_numpy(x).cuda()[1:]          # 4-byte offset: no TMA tensor map
    assert xd.data_ptr() % 16 != 0
    p = H.QuantParams(0.01, (n,), 32, "f32")
    s = H.compress(H.RawArray(xd, (n,), "f32"), p)
    ref = O.compress(x[1:], 0.01, (n,), 32, "f32")
    assert H.serialize(s.to_host()) == O.serialize(ref)


def test_compress_exact_tiles_mixed(H):
    """bins beyond 2^30 in some tiles only: exact tiles interleave with
    register tiles in the look-back chain"""
    # f32 data can reach |bin| >= 2^30 only on the grid itself (otherwise the
    # reference raises the resolution error): integer values at eps = 0.5
    n = 4096 * 12
    rng = np.random.default_rng(3)
    x = np.round(rng.normal(0, 50, n)).astype(np.float32)
    x[4096 * 3:4096 * 4] = (rng.integers(-2 ** 20, 2 ** 20, 4096) * 1536).astype(np.float32)  # |bin| < 2^31
    x[4096 * 9 + 100] = 1.5 * 2.0 ** 30          # one element in tile 9
    _full_check(H, x, 0.5, (n,))


def test_compress_resolution_error_class(H):
    n = 4096 * 4
    x = np.random.default_rng(1).normal(0, 1e4, n).astype(np.float32)
    with pytest.raises(H.QuantOverflow):
        H.compress(H.RawArray(x, (n,), "f32"), H.QuantParams(1e-6, (n,), 32, "f32"))
    with pytest.raises(O.QuantOverflow):
        O.compress(x, 1e-6, (n,), 32, "f32")


def test_compress_certificate_margin(H):
    """values placed exactly on / next to bin edges (x = (2k+1) eps - eps)"""
    eps = 0.0123456789
    k = np.arange(-50000, 50000, dtype=np.float64)
    edges = (2.0 * k) * eps                       # (x + eps) / 2eps = k + 1/2 ... edges of floor
    x = np.concatenate([edges, np.nextafter(edges.astype(np.float32), np.inf).astype(np.float64),
                        np.nextafter(edges.astype(np.float32), -np.inf).astype(np.float64),
                        (2.0 * k + 1.0) * eps]).astype(np.float32)
    _full_check(H, x, eps, (x.size,))


def _bins_stream(H, bins, n):
    p = H.QuantParams(0.01, (n,), 32, "f32")
    s = H.encode_from_quant(H.QuantArray(bins, p))
    ref = O.encode_bins(bins, 0.01, (n,), 32, "f32")
    _check_stream(H, s, ref)
    return s, ref


@pytest.mark.parametrize("hi", [2 ** 20, 2 ** 27, 2 ** 31 - 1])
def test_decode_wide_and_unstaged_tiles(H, hi):
    """widths > 24 (exact decode), tiles with > 16 KB of payload (in place)"""
    n = 4096 * 6 + 13
    rng = np.random.default_rng(hi % 1000)
    bins = rng.integers(-hi, hi, n)
    bins[: 4096 * 2] = rng.integers(-50, 50, 4096 * 2)      # ordinary register tiles too
    s, ref = _bins_stream(H, bins, n)
    assert np.array_equal(H.decode_to_quant(s).bins, bins)
    assert H.decompress(s).values.tobytes() == O.decompress(ref).tobytes()
    S, Q = O.moments(ref)
    assert H.mean(s) == O.mean_from(S, n, 0.01)
    assert H.variance(s) == O.variance_from(S, Q, n, 0.01)


@pytest.mark.parametrize("scalar", [-1.25, 3.0e5, -7.7e6, 4.3e8])
def test_scalar_mul_paths(H, scalar):
    """|rs| < 2^23 register path, larger scalars exact path, overflow classes"""
    n = 4096 * 5 + 9
    rng = np.random.default_rng(11)
    bins = np.cumsum(rng.integers(-40, 40, n))
    bins[4096:4096 + 64] = rng.integers(-2 ** 29, 2 ** 29, 64)   # big outliers in one tile
    s, ref = _bins_stream(H, bins, n)
    try:
        want = O.serialize(O.scalar_mul(ref, scalar))
    except O.OracleError as exc:
        with pytest.raises(H.HoszpError) as ei:
            H.scalar_mul(s, scalar)
        assert type(ei.value).__name__ == type(exc).__name__
    else:
        assert H.serialize(H.scalar_mul(s, scalar)) == want


def test_chain_device_resident_matches_host(H):
    """the device-resident chain (no host round trips between ops) equals the
    oracle's chain byte for byte"""
    import torch

    n = 4096 * 30 + 17
    rng = np.random.default_rng(5)
    x = (np.sin(np.arange(n) / 500.0) * 30 + rng.normal(0, 0.05, n)).astype(np.float32)
    raw = H.RawArray(torch.from_numpy(x).cuda(), (n,), "f32")
    eps = H.resolve_eps(raw, 1e-4, "rel")
    p = H.QuantParams(eps, (n,), 32, "f32")
    z = H.scalar_mul(H.scalar_add(H.negate(H.compress(raw, p)), 3.5), -1.25)
    zr = O.scalar_mul(O.scalar_add(O.negate(O.compress(x, eps, (n,), 32, "f32")), 3.5), -1.25)
    assert H.serialize(z.to_host()) == O.serialize(zr)
    S, Q = O.moments(zr)
    assert H.mean(z) == O.mean_from(S, n, eps)
    assert H.variance(z) == O.variance_from(S, Q, n, eps)
    assert H.decompress(z).values.cpu().numpy().tobytes() == O.decompress(zr).tobytes()


def test_compress_wide_tiles_mixed(H):
    """Float32 fields whose tiles mix register-path blocks with blocks whose
    bins reach 2^30 (the compressor's exact warp-per-block path places those
    tiles itself): stream bytes against the oracle, and the bins re-encode to
    the same bytes."""
    import torch

    import hoszp_oracle as O

    rng = np.random.default_rng(5)
    for _ in range(6):
        n = 4096 * int(rng.integers(2, 12)) + int(rng.integers(0, 40))
        x = (rng.normal(0, 1, n) * 10 + 100).astype(np.float32)
        for t in rng.choice(n // 4096, size=max(1, n // 8192), replace=False):
            x[t * 4096 + 5: t * 4096 + 300: 7] = 3.0e6      # bins ~1.5e9 inside blocks
        p = H.QuantParams(1e-3, (n,), 32, "f32")
        s = H.compress(H.RawArray(torch.from_numpy(x).cuda(), (n,), "f32"), p)
        want = O.serialize(O.compress(x, 1e-3, (n,), 32, "f32"))
        assert H.serialize(s.to_host()) == want
        assert H.serialize(H.encode_from_quant(H.decode_to_quant(s)).to_host()) == want


@pytest.mark.parametrize("w", [17, 20, 22, 24])
def test_moments_monotone_wide_residuals(H, w):
    """Register-path block sums at the widest register widths with same-sign
    residuals: sum_i P_i reaches 496 * 2^w (beyond int32 for w >= 22)."""
    n = 4096 * 4 + 45
    rng = np.random.default_rng(w)
    d = rng.integers(1 << (w - 1), 1 << w, n).astype(np.int64)
    blk = np.arange(n) // 32
    d *= rng.choice([-1, 1], blk[-1] + 1)[blk]                 # rising and falling ramps
    d[::32] = rng.integers(-(1 << 28), 1 << 28, d[::32].size)   # block starts: the outliers
    bins = np.zeros(n, dtype=np.int64)
    for b in range(blk[-1] + 1):                               # per-block ramps
        sl = slice(32 * b, min(32 * b + 32, n))
        bins[sl] = np.cumsum(d[sl])
    s, ref = _bins_stream(H, bins, n)
    assert int(np.asarray(ref["widths"]).max()) == w
    S, Q = O.moments(ref)
    assert H.mean(s) == O.mean_from(S, n, 0.01)
    assert H.variance(s) == O.variance_from(S, Q, n, 0.01)
    assert np.array_equal(H.decode_to_quant(s).bins, bins)


def test_prefetch_totals_matches_fetch(H):
    """DeviceStream.prefetch_totals (side-stream copy into the pinned ring)
    gives the same totals as the synchronous fetch, also when the ring wraps
    around before the value is read."""
    import torch

    from paper_2408_11971_b200.device import DeviceStream

    n = 4096 * 5 + 3
    rng = np.random.default_rng(5)
    x = torch.from_numpy(np.cumsum(rng.normal(0, 1, n)).astype(np.float32)).cuda()
    p = H.QuantParams(0.01, (n,), 32, "f32")
    streams = [H.compress(H.RawArray(x * (1 + i), (n,), "f32"), p) for i in range(3)]
    want = []
    for s in streams:
        hs = s.to_host()
        want.append((len(hs.sign_planes), len(hs.payload)))
    fresh = [DeviceStream.from_host(s.to_host()) for s in streams]
    for s in fresh:
        s._totals = None
        s.prefetch_totals()
    assert [s.totals() for s in fresh] == want
    # wrap the ring (64 slots) before reading the first prefetch: falls back
    first = DeviceStream.from_host(streams[0].to_host())
    first._totals = None
    first.prefetch_totals()
    for _ in range(70):
        d = DeviceStream.from_host(streams[1].to_host())
        d._totals = None
        d.prefetch_totals()
    assert first.totals() == want[0] and d.totals() == want[1]


@pytest.mark.parametrize("n,kind", [(4096, "small"), (4096 * 3 + 17, "small"), (4096 * 64 + 31, "edge"),
                                    (4096 * 40 + 5, "mixed"), (32 * 5000, "huge"),
                                    (4096 * 8, "tailless_wide")])
def test_encode_from_quant_register_path(H, n, kind):
    """encode_from_quant for block_len 32 runs on the compressor's register
    encoder (int64 bin tiles by a 3-D TMA load); tiles holding a bin with
    |bin| >= 2^30 take the exact path.  Bytes against the oracle's
    encode_bins (codec.py:523-525), round trip through decode_to_quant."""
    rng = np.random.default_rng(n)
    if kind == "small":
        bins = np.cumsum(rng.integers(-40, 41, n)).astype(np.int64)
    elif kind == "edge":               # |bin| right at the register-path limit 2^30
        bins = rng.integers(-(2 ** 30 - 1), 2 ** 30, n).astype(np.int64)
        bins[rng.integers(0, n, 20)] = 2 ** 30 - 1
        bins[rng.integers(0, n, 20)] = -(2 ** 30 - 1)
    elif kind == "mixed":              # a few wide tiles among narrow ones
        bins = rng.integers(-1000, 1000, n).astype(np.int64)
        for t in (3, 17, 31):
            bins[t * 4096 + 7] = 2 ** 30
            bins[t * 4096 + 100] = -(2 ** 40)
    elif kind == "huge":               # 62-bit bins: widths 63-64, the exact path everywhere
        bins = rng.integers(-(2 ** 62), 2 ** 62, n).astype(np.int64)
        bins[::32] = rng.integers(-1000, 1000, bins[::32].size)   # outliers stay int32
    else:
        bins = rng.integers(-(2 ** 31), 2 ** 31, n).astype(np.int64)
    p = H.QuantParams(0.5, (n,), 32, "f32")
    s = H.encode_from_quant(H.QuantArray(bins, p))
    ref = O.encode_bins(bins, p.eps, p.dims, p.block_len, p.dtype)
    assert H.serialize(s) == O.serialize(ref)
    assert np.array_equal(H.decode_to_quant(s).bins, bins)


def _alternating_width_bins(n, w_small, w_big, seed):
    """Bins whose tiles alternate between residual widths w_small and w_big:
    residuals of exactly w bits with alternating signs, so |bin| stays below
    1000 + 2^w."""
    rng = np.random.default_rng(seed)
    bins = np.empty(n, dtype=np.int64)
    for t in range(-(-n // 4096)):
        w = w_big if t % 2 else w_small
        seg = bins[t * 4096:(t + 1) * 4096]
        mag = rng.integers(2 ** (w - 1), 2 ** w, seg.size)
        d = np.where(np.arange(seg.size) % 2 == 0, mag, -mag)
        d[::32] = 0
        seg[:] = rng.integers(-1000, 1000)
        full = seg.size // 32 * 32
        seg[:full].reshape(-1, 32)[:] += np.cumsum(d[:full].reshape(-1, 32), axis=1)
        seg[full:] += np.cumsum(d[full:])
    return bins


@pytest.mark.parametrize("w_small,w_big", [(12, 24), (10, 27), (12, 21), (11, 22)])
def test_encoder_ring_small_then_large_tile(H, w_small, w_big):
    """Staging-ring regression: a CTA that packs a small tile and then a large
    one skips the rest of its 16 KB ring; the skipped bytes belong to no tile,
    and the free-space wait used to count them as occupied forever (a tile
    followed by a larger one of more than the space left hung compress and
    encode_from_quant: 128 * 4 * (w_small + w_big) > 16384).  Tiles alternate
    between the two residual widths; bytes against the oracle for
    encode_from_quant and, where float32 holds the bins exactly, compress."""
    n = 4096 * 1600 + 11        # more tiles than resident CTAs: every CTA packs several
    bins = _alternating_width_bins(n, w_small, w_big, w_small * 100 + w_big)
    assert np.abs(bins).max() < 2 ** 30
    p = H.QuantParams(0.5, (n,), 32, "f32")
    ref = O.encode_bins(bins, p.eps, p.dims, p.block_len, p.dtype)
    assert {w_small, w_big} <= set(int(v) for v in ref["widths"])
    s = H.encode_from_quant(H.QuantArray(bins, p))
    assert H.serialize(s) == O.serialize(ref)
    if w_big <= 22:
        # x = bin exactly (|bin| < 2^24); eps 0.5: floor((x + 0.5) / 1) = bin
        x = bins.astype(np.float32)
        assert np.array_equal(x.astype(np.int64), bins)
        sc = H.compress(H.RawArray(x, (n,), "f32"), p)
        assert H.serialize(sc) == O.serialize(O.compress(x, 0.5, (n,), 32, "f32"))
        assert H.serialize(sc) == O.serialize(ref)


def test_scalar_mul_overflow_detected_after_input_release(H):
    """scalar_mul releases the staged input tile right after the decode; a tile
    whose RESCALED bins leave the register range (|bin'| >= 2^30) is only
    detected afterwards and re-decodes from global memory with the header
    copies kept outside the staged tile.  Tiles alternate between bins that
    stay in range and bins that leave it; many more tiles than resident CTAs,
    so every CTA meets both kinds back to back.  Bytes against the oracle."""
    ntiles = 1500
    n = 4096 * ntiles + 5
    rng = np.random.default_rng(77)
    bins = np.cumsum(rng.integers(-3, 4, n)).astype(np.int64)
    big = (np.arange(n) // 4096) % 3 == 1
    bins[big] += 40_000_000                       # x 30 -> 1.2e9 >= 2^30
    s, ref = _bins_stream(H, bins, n)
    scalar = 30.0                                  # eps 0.01: rs = 1500 (< 2^23), bin' = round(0.02 * 1500 * bin)
    want = O.scalar_mul(ref, scalar)
    got = H.scalar_mul(s, scalar)
    assert H.serialize(got) == O.serialize(want)
    # and the same stream device-resident (asynchronous path)
    ds = H.DeviceStream.from_host(s)
    assert H.serialize(H.scalar_mul(ds, scalar).to_host()) == O.serialize(want)


@pytest.mark.parametrize("bad", [float("nan"), float("inf"), -float("inf")])
def test_compress_unvalidated_nonfinite_is_flagged(H, bad):
    """The compressor tests its float32 certificate once per 32-element row, on
    the smallest |v| and the largest |p| of the row; the maximum propagates
    NaN, so a non-finite value that skipped RawArray's finite check (a
    pre-validated array) still fails the test and reaches the exact
    quantizer, which reports it like the reference's 63-bit guard
    (codec.py:136-137)."""
    import torch

    n = 4096 * 3 + 7
    x = torch.linspace(-5.0, 5.0, n, device="cuda", dtype=torch.float32)
    x[4096 + 777] = bad
    raw = H.RawArray(x, (n,), "f32", _validated=True)
    with pytest.raises(H.QuantOverflow):
        H.compress(raw, H.QuantParams(1e-3, (n,), 32, "f32")).check()
