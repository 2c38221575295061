"""Config 5 slab scale (2^30 values, 4 GiB of float32 -- the per-GPU shard
of the 2048^3 field at 8 GPUs): the whole path at full size, checked through
size-independent properties plus an oracle comparison of a block-aligned
prefix (a stream's sections for a block range are self-contained, so the
prefix of the big stream must equal the oracle's stream of the prefix)."""

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


def test_config5_slab_full_size(H):
    import torch

    from paper_2408_11971_b200 import workloads as W

    x = W.config5_slab(0)                                  # 2^30 f32 on the device
    n = x.numel()
    assert n == 1 << 30
    c = W.CONFIGS[5]
    raw = H.RawArray(x, (n,), "f32")
    eps = H.resolve_eps(raw, c["rel_eps"], "rel")
    p = H.QuantParams(eps, (n,), 32, "f32")
    s = H.compress(raw, p)
    sb, pb = s.totals()
    assert sb + pb < 4 * n

    # block-aligned prefix == the oracle's stream of the prefix
    m = 32 * 40_000
    ref = O.compress(x[:m].cpu().numpy(), eps, (m,), 32, "f32")
    nb = m // 32
    assert s.widths[:nb].cpu().numpy().tobytes() == ref["widths"].tobytes()
    assert np.array_equal(s.outliers[:nb].cpu().numpy(), ref["outliers"])
    assert s.signs[:len(ref["signs"])].cpu().numpy().tobytes() == ref["signs"]
    assert s.payload[:len(ref["payload"])].cpu().numpy().tobytes() == ref["payload"]

    # error bound of the reconstruction (codec.py:150-154, then f32 rounding)
    y = H.decompress(s).values
    err = (y.double() - x.double()).abs().max().item()
    ulp = float(np.spacing(np.float32(x.abs().max().item())))
    assert err <= eps * (1 + 1e-9) + ulp

    # mean / variance within 1e-12 relative of float64 statistics of the grid
    g = H.decompress(s, out_dtype=np.float64).values
    mu, var = H.mean(s), H.variance(s)
    assert abs(mu - g.mean().item()) <= 1e-12 * abs(mu)
    assert abs(var - g.var(unbiased=False).item()) <= 1e-10 * var

    # homomorphic identities at full size
    nn = H.negate(H.negate(s))
    assert torch.equal(nn.signs[:sb], s.signs[:sb]) and torch.equal(nn.outliers, s.outliers)
    z = H.elementwise_add(s, H.negate(s))
    assert int(z.widths.max().item()) == 0 and int(z.outliers.abs().max().item()) == 0
    t = H.scalar_mul(H.scalar_add(s, 3.5), -1.25)
    assert t.totals()[1] > 0
    del y, g
