"""Full-size BASELINE configs 1-4: the GPU pipeline against the CPU oracle on
the same seeded field, bit-exact (stream bytes, decoded values, transformed
streams, exact mean/variance).  Config 5 (2^33 values) is covered per slab in
test_gpu_sharding.py.
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


def _pipeline(H, x, dims, rel, sadd, smul, full_oracle=True):
    raw = H.RawArray(x, dims, "f32")
    eps = H.resolve_eps(raw, rel, "rel")
    assert eps == O.resolve_eps(x, rel, "rel")
    p = H.QuantParams(eps, dims, 32, "f32")
    s = H.compress(raw, p)
    ref = O.compress(x, eps, dims, 32, "f32")
    assert H.serialize(s) == O.serialize(ref), "compress"
    assert H.decompress(s).values.tobytes() == O.decompress(ref).tobytes(), "decompress"
    S, Q = O.moments(ref)
    n = x.size
    assert H.mean(s) == O.mean_from(S, n, eps)
    assert H.variance(s) == O.variance_from(S, Q, n, eps)
    z = H.negate(s)
    zr = O.negate(ref)
    assert H.serialize(z) == O.serialize(zr), "negate"
    z = H.scalar_add(z, sadd)
    zr = O.scalar_add(zr, sadd)
    assert H.serialize(z) == O.serialize(zr), "scalar_add"
    if full_oracle:
        z = H.scalar_mul(z, smul)
        zr = O.scalar_mul(zr, smul)
        assert H.serialize(z) == O.serialize(zr), "scalar_mul"
        S, Q = O.moments(zr)
        assert H.mean(z) == O.mean_from(S, n, eps)
        assert H.variance(z) == O.variance_from(S, Q, n, eps)
        assert H.decompress(z).values.tobytes() == O.decompress(zr).tobytes()
    return s


def test_config1_pipeline(H):
    from paper_2408_11971_b200 import workloads as W

    c = W.CONFIGS[1]
    _pipeline(H, W.config1(), c["dims"], c["rel_eps"], c["sadd"], c["smul"])


def test_config2_all_ops(H):
    from paper_2408_11971_b200 import workloads as W

    c = W.CONFIGS[2]
    _pipeline(H, W.config2(), c["dims"], c["rel_eps"], c["sadd"], c["smul"])


@pytest.mark.parametrize("rel", [1e-3, 1e-4, 1e-5])
def test_config3_sweep(H, rel):
    from paper_2408_11971_b200 import workloads as W

    c = W.CONFIGS[3]
    s = _pipeline(H, W.config3(), c["dims"], rel, c["sadd"], c["smul"])
    assert (s.widths == 0).mean() > 0.2          # constant blocks exercised


def test_config4_all_ops(H):
    from paper_2408_11971_b200 import workloads as W

    c = W.CONFIGS[4]
    x = W.config4(device="cuda").cpu().numpy()
    s = _pipeline(H, x, c["dims"], c["rel_eps"], c["sadd"], c["smul"])
    assert int(s.widths.max()) >= 8
