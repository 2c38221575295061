"""The drop-in boundary: the C-ABI library loads without a GPU and exports
every symbol include/hsz_b200.h declares, with the documented host-only
geometry helpers behaving as specified.  (No compute calls here.)"""

import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "hsz_b200.h")


def _declared():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(hsz_[a-z0-9_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    from paper_2408_11971_b200 import _native

    return _native.load()


def test_header_declares_the_hot_path():
    names = _declared()
    for must in ("hsz_compress", "hsz_decode", "hsz_negate", "hsz_scalar_add", "hsz_scalar_mul",
                 "hsz_moments", "hsz_minmax", "hsz_tile_offsets", "hsz_encode_bins",
                 "hsz_elementwise"):
        assert must in names


def test_every_declared_symbol_is_exported(lib):
    for name in _declared():
        assert hasattr(lib, name), name


def test_ctypes_binding_covers_the_header():
    from paper_2408_11971_b200 import _native

    assert sorted(_native.SIGNATURES) == _declared()


def test_version(lib):
    assert lib.hsz_version().startswith(b"hsz_b200")


def test_geometry_helpers(lib):
    # B = ceil(n / k), tiles of 128 blocks (model.py:81-84)
    assert lib.hsz_tile_count(1, 32) == 1
    assert lib.hsz_tile_count(128 * 32, 32) == 1
    assert lib.hsz_tile_count(128 * 32 + 1, 32) == 2
    assert lib.hsz_tile_count(25_000_000, 32) == -(-781_250 // 128)
    # worst-case sections: ceil(k/8) sign bytes and 8k payload bytes per block
    assert lib.hsz_sign_bound(100, 33) == 4 * 5
    assert lib.hsz_payload_bound(100, 32) == 4 * 256
    assert lib.hsz_scalar_mul_scratch_size(1000, 32) == 0
    assert lib.hsz_scalar_mul_scratch_size(1000, 33) == 8000
    ws = lib.hsz_workspace_size(25_000_000, 32)
    assert ws >= 8 * 7 * lib.hsz_tile_count(25_000_000, 32)


def test_argument_errors_do_not_touch_the_gpu(lib):
    # invalid arguments are rejected before any CUDA call (HSZ_EINVAL = -1)
    assert lib.hsz_compress(None, 0, 10, 32, 0.1, None, None, None, 0, None, 0, None, None,
                            None, 0, None) == -1
    assert lib.hsz_decode(None, None, None, None, None, 10, 32, 0.1, 0, None, None, None) == -1
    assert lib.hsz_scalar_add(None, None, 0, 1, None, None) == -1
    z = [None] * 10
    assert lib.hsz_elementwise(*z, 10, 32, 0, None, None, None, 0, None, 0, None, None, None, None,
                               0, None) == -1
    assert lib.hsz_hadamard(*z, 10, 32, 0.1, None, None, None, 0, None, 0, None, None, None, None,
                            0, None) == -1
    assert lib.hsz_pair_stats(*z, 10, 32, None, None, None, None) == -1
    assert lib.hsz_block_means(None, None, None, None, None, 10, 32, 0.1, None, None, None,
                               None) == -1
    assert lib.hsz_moments_mb(None, None, None, None, None, 10, 32, 0, None, None, None, 0, None, 1,
                              None) == -1
    assert lib.hsz_minmax_mb(None, 0, 10, None, None, None, 0, None, 1, None) == -1


def test_scratch_queries(lib):
    assert lib.hsz_elementwise_scratch_size(1000, 32) == 0        # one fused pass
    assert lib.hsz_elementwise_scratch_size(1000, 33) == 8000
    assert lib.hsz_bivariate_scratch_size(1000, 32) == 16000
