"""GPU parity of the element-wise operations on two compressed streams
(reference ops.py:163-192) through the C ABI: against the reference's own
outputs (tests/golden/golden_elementwise.npz, made by
tests/golden/make_golden_elementwise.py) and against the CPU oracle on
seeded fields at the B200 fast-path sizes.  Bit-exact stream bytes.
"""

import os

import numpy as np
import pytest

import hoszp_oracle as O

pytestmark = pytest.mark.gpu

_Z = np.load(os.path.join(os.path.dirname(__file__), "golden", "golden_elementwise.npz"))
_N = int(_Z["count"][0])


@pytest.fixture(scope="module")
def H():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2408_11971_b200 as mod

    return mod


@pytest.mark.parametrize("case", range(_N))
def test_elementwise_golden(H, case):
    a = H.deserialize(_Z[f"c{case}_a"].tobytes())
    b = H.deserialize(_Z[f"c{case}_b"].tobytes())
    for name, fn in (("add", H.elementwise_add), ("sub", H.elementwise_sub)):
        err = str(_Z[f"c{case}_{name}_err"][0])
        if err:
            with pytest.raises(Exception) as ei:
                fn(a, b)
            assert type(ei.value).__name__ == err
            continue
        got = fn(a, b)
        assert H.serialize(got) == _Z[f"c{case}_{name}"].tobytes(), name
        # the dispatch table reaches the same kernel
        got2 = H.apply_stream_op("eadd" if name == "add" else "esub", [a, b])
        assert H.serialize(got2) == H.serialize(got)


def _field(rng, n, kind):
    i = np.arange(n)
    if kind == 0:
        return (np.sin(i / 700.0) * 40 + 280 + rng.normal(0, 0.3, n)).astype(np.float32)
    if kind == 1:
        x = rng.normal(0, 5, n).astype(np.float32)
        x[(i // 4096) % 3 == 0] = 2.5                       # constant blocks
        return x
    return np.exp(rng.normal(0, 1.5, n)).astype(np.float32)   # heavy tail, wide blocks


@pytest.mark.parametrize("n,kind,rel", [(4096 * 40 + 13, 0, 1e-4), (4096 * 64, 1, 1e-3),
                                        (300_001, 2, 1e-5), (1 << 20, 0, 1e-3)])
def test_elementwise_device_chain(H, n, kind, rel):
    """Device-resident operands (compressed on the GPU), a +/- b compared with
    the oracle on the same streams; also (a - b) + b == a byte for byte."""
    import torch

    rng = np.random.default_rng(n + kind)
    xa, xb = _field(rng, n, kind), _field(rng, n, (kind + 1) % 3)
    lo = float(min(xa.min(), xb.min()))
    hi = float(max(xa.max(), xb.max()))
    p = H.QuantParams(rel * (hi - lo), (n,), 32, "f32")
    sa = H.compress(H.RawArray(torch.from_numpy(xa).cuda(), (n,), "f32"), p)
    sb = H.compress(H.RawArray(torch.from_numpy(xb).cuda(), (n,), "f32"), p)
    ha, hb = sa.to_host(), sb.to_host()
    oa, ob = O.deserialize(H.serialize(ha)), O.deserialize(H.serialize(hb))
    add = H.elementwise_add(sa, sb)
    sub = H.elementwise_sub(sa, sb)
    assert H.serialize(add.to_host()) == O.serialize(O.elementwise_add(oa, ob))
    assert H.serialize(sub.to_host()) == O.serialize(O.elementwise_sub(oa, ob))
    back = H.elementwise_add(sub, sb)
    assert H.serialize(back.to_host()) == H.serialize(ha)


def test_elementwise_params_mismatch(H):
    p1 = H.QuantParams(0.01, (64,), 32, "f32")
    p2 = H.QuantParams(0.01, (64,), 16, "f32")
    a = H.encode_from_quant(H.QuantArray(np.arange(64, dtype=np.int64), p1))
    b = H.encode_from_quant(H.QuantArray(np.arange(64, dtype=np.int64), p2))
    with pytest.raises(H.ParamsMismatch):
        H.elementwise_add(a, b)


@pytest.mark.parametrize("j", range(int(_Z["agg_count"][0])))
def test_aggregate_golden(H, j):
    """N-way homomorphic aggregation (distsim.py:80-103) against the
    reference's own output, host and device-resident operands."""
    from paper_2408_11971_b200 import distsim

    cnt = int(_Z[f"agg{j}_count"][0])
    ss = [H.deserialize(_Z[f"agg{j}_in{m}"].tobytes()) for m in range(cnt)]
    want = _Z[f"agg{j}_out"].tobytes()
    assert H.serialize(distsim.aggregate_homomorphic(ss)) == want
    dev = [H.DeviceStream.from_host(s) for s in ss]
    assert H.serialize(distsim.aggregate_homomorphic(dev).to_host()) == want


def _float_or_err(fn):
    try:
        return fn().hex()
    except Exception as exc:
        return "!" + type(exc).__name__


@pytest.mark.parametrize("case", range(_N))
def test_bivariate_golden(H, case):
    """hadamard / covariance / ssim_global / block_means through the C ABI
    against the reference's own outputs (bit-exact bytes and floats)."""
    a = H.deserialize(_Z[f"c{case}_a"].tobytes())
    b = H.deserialize(_Z[f"c{case}_b"].tobytes())
    err = str(_Z[f"c{case}_had_err"][0])
    if err:
        with pytest.raises(Exception) as ei:
            H.hadamard(a, b)
        assert type(ei.value).__name__ == err
    else:
        assert H.serialize(H.hadamard(a, b)) == _Z[f"c{case}_had"].tobytes()
    assert _float_or_err(lambda: H.covariance(a, b)) == str(_Z[f"c{case}_cov"][0])
    assert _float_or_err(lambda: H.ssim_global(a, b)) == str(_Z[f"c{case}_ssim"][0])
    assert H.block_means(a).tobytes() == _Z[f"c{case}_bmeans"].tobytes()
    if not str(_Z[f"c{case}_cov"][0]).startswith("!"):
        assert H.apply_reduction("covariance", [a, b]).hex() == str(_Z[f"c{case}_cov"][0])


def test_bivariate_device_resident(H):
    """Device-resident operands at a realistic size against the oracle."""
    import torch

    rng = np.random.default_rng(77)
    n = 300_000 + 11
    xa, xb = _field(rng, n, 0), _field(rng, n, 1)
    p = H.QuantParams(1e-3 * float(max(xa.max(), xb.max()) - min(xa.min(), xb.min())), (n,), 32, "f32")
    sa = H.compress(H.RawArray(torch.from_numpy(xa).cuda(), (n,), "f32"), p)
    sb = H.compress(H.RawArray(torch.from_numpy(xb).cuda(), (n,), "f32"), p)
    oa = O.deserialize(H.serialize(sa.to_host()))
    ob = O.deserialize(H.serialize(sb.to_host()))
    assert H.serialize(H.hadamard(sa, sb).to_host()) == O.serialize(O.hadamard(oa, ob))
    assert H.covariance(sa, sb) == O.covariance(oa, ob)
    assert H.ssim_global(sa, sb) == O.ssim_global(oa, ob)
    assert H.block_means(sa).cpu().numpy().tobytes() == O.block_means(oa).tobytes()


def _wide_bins(case, n, rng):
    """Operand bins whose residuals are ~2^63 (widths 63-64): their BIN sums
    leave int64, their residual sums do not fit 63 bits."""
    A = (1 << 62) - 1
    a = np.where(np.arange(n) % 2 == 0, A, -A).astype(np.int64)
    a[::32] = rng.integers(-1000, 1000, a[::32].size)
    if case == "self":
        b = a.copy()                      # residual sums ~2^64 - 4: width 64
    elif case == "neg":
        b = -a                            # everything cancels: width 0
    else:
        b = a.copy()
        b[1::2] = rng.integers(-(1 << 40), 1 << 40, b[1::2].size)
    return a, b


@pytest.mark.parametrize("case", ["self", "neg", "mixed"])
@pytest.mark.parametrize("sub", [False, True])
def test_elementwise_wide_operands_residual_domain(H, case, sub):
    """the element-wise exact path combines RESIDUALS (128-bit),
    like the reference (ops.py:163-182, Python ints past int64), instead of
    bins modulo 2^64 -- operands of width 62-64 give the reference's stream,
    not a spurious QuantOverflow or a wrapped sign."""
    rng = np.random.default_rng(7)
    n = 32 * 4 * 3 + 5
    a, b = _wide_bins(case, n, rng)
    if sub:
        b = -b
    oa = O.encode_bins(a, 0.5, (n,), 32, "f32")
    ob = O.encode_bins(b, 0.5, (n,), 32, "f32")
    want = O.elementwise_sub(oa, ob) if sub else O.elementwise_add(oa, ob)
    ha, hb = H.deserialize(O.serialize(oa)), H.deserialize(O.serialize(ob))
    got = H.elementwise_sub(ha, hb) if sub else H.elementwise_add(ha, hb)
    assert H.serialize(got) == O.serialize(want)
