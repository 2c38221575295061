"""Host-side contract: the model / byte layout mirror against the reference
goldens (FORMAT.md, pkg/tests/test_model.py) and the error-word mapping."""

import numpy as np
import pytest

import hoszp_oracle as O
import paper_2408_11971_b200 as H
from paper_2408_11971_b200 import errors as E
from conftest import EXAMPLE_HEX, load_golden

CASES = load_golden()


def _example_stream():
    p = H.QuantParams(0.01, (2, 2), 32, "f32")
    return H.CompressedStream(p, np.array([2]), np.array([-1]), b"\x20", b"\x08")


def test_format_md_dump():
    assert H.serialize(_example_stream()) == bytes.fromhex(EXAMPLE_HEX)
    assert H.deserialize(bytes.fromhex(EXAMPLE_HEX)) == _example_stream()


@pytest.mark.parametrize("case", [c for c in CASES if not c.s("err")], ids=repr)
def test_golden_round_trip(case):
    s = H.deserialize(case.bytes_of("stream"))
    assert s.params == H.QuantParams(case.eps, case.dims, case.block_len, case.dtype)
    assert H.serialize(s) == case.bytes_of("stream")
    ref = O.encode_bins(case["bins_out"], case.eps, case.dims, case.block_len, case.dtype)
    assert np.array_equal(s.widths, ref["widths"])
    assert s.sign_planes == ref["signs"] and s.payload == ref["payload"]


class TestParams:                                       # test_model.py:12-60
    def test_defaults(self):
        p = H.QuantParams(0.5, (4, 5))
        assert p.block_len == 32 and p.dtype == "f32"
        assert p.element_count == 20 and p.block_count == 1

    @pytest.mark.parametrize("bad", [dict(eps=0.0), dict(eps=float("inf")), dict(dims=()),
                                     dict(dims=(0,)), dict(block_len=0), dict(dtype="f16")])
    def test_rejects(self, bad):
        kw = dict(eps=0.1, dims=(4,), block_len=32, dtype="f32")
        kw.update(bad)
        with pytest.raises(ValueError):
            H.QuantParams(**kw)

    def test_block_lengths_tail(self):
        p = H.QuantParams(0.1, (70,), 32)
        assert list(p.block_lengths()) == [32, 32, 6]


class TestStreamChecks:                                 # test_model.py:90-119
    def test_size_cross_checks(self):
        s = _example_stream()
        with pytest.raises(H.GeometryMismatch):
            H.CompressedStream(s.params, s.widths, s.outliers, b"", s.payload)
        with pytest.raises(H.GeometryMismatch):
            H.CompressedStream(s.params, s.widths, s.outliers, s.sign_planes, s.payload + b"\0")
        with pytest.raises(H.GeometryMismatch):
            H.CompressedStream(s.params, np.array([65]), s.outliers, b"\0", b"\0" * 33)

    def test_outlier_guard(self):
        s = _example_stream()
        with pytest.raises(H.OutlierOverflow):
            H.CompressedStream(s.params, s.widths, np.array([2 ** 31]), s.sign_planes, s.payload)

    def test_serialized_size_and_ratio(self):
        s = _example_stream()
        assert s.serialized_size == 43
        assert s.compression_ratio == pytest.approx(16 / 43)


class TestDeserializeErrors:                            # test_model.py:184-228
    def test_bad_magic(self):
        with pytest.raises(H.BadMagic):
            H.deserialize(b"XXXX" + bytes.fromhex(EXAMPLE_HEX)[4:])
        with pytest.raises(H.BadMagic):
            H.deserialize(b"HX")

    def test_truncated(self):
        raw = bytes.fromhex(EXAMPLE_HEX)
        for cut in (3, 10, 25, 37, 41, 42):
            with pytest.raises(H.FormatError):
                H.deserialize(raw[:cut])

    def test_version(self):
        raw = bytearray.fromhex(EXAMPLE_HEX)
        raw[4] = 2
        with pytest.raises(H.VersionMismatch):
            H.deserialize(bytes(raw))

    def test_trailing_bytes(self):
        with pytest.raises(H.GeometryMismatch):
            H.deserialize(bytes.fromhex(EXAMPLE_HEX) + b"\0")


class TestErrorWord:
    @pytest.mark.parametrize("bits,cls", [
        (E.ERR_NONFINITE, ValueError), (E.ERR_QUANT_OVERFLOW, H.QuantOverflow),
        (E.ERR_QUANT_RESOLUTION, H.QuantOverflow), (E.ERR_PREFIX_OVERFLOW, H.QuantOverflow),
        (E.ERR_RESCALE_OVERFLOW, H.QuantOverflow), (E.ERR_OUTLIER_OVERFLOW, H.OutlierOverflow),
        (E.ERR_BAD_WIDTH, H.GeometryMismatch), (E.ERR_OUTPUT_NONFINITE, ValueError)])
    def test_mapping(self, bits, cls):
        with pytest.raises(cls):
            E.raise_for_flags(bits)

    def test_precedence_follows_the_reference_stage_order(self):
        # prefix overflow (decode) is raised before the int32 guard (re-encode)
        with pytest.raises(H.QuantOverflow):
            E.raise_for_flags(E.ERR_PREFIX_OVERFLOW | E.ERR_OUTLIER_OVERFLOW)
        E.raise_for_flags(0)

    def test_header_bits_match(self):
        import os
        import re

        hdr = open(os.path.join(os.path.dirname(os.path.dirname(__file__)), "include",
                                "hsz_b200.h")).read()
        for name in ("NONFINITE", "QUANT_OVERFLOW", "QUANT_RESOLUTION", "PREFIX_OVERFLOW",
                     "RESCALE_OVERFLOW", "OUTLIER_OVERFLOW", "CAPACITY", "OUTPUT_NONFINITE",
                     "BAD_WIDTH"):
            m = re.search(rf"#define HSZ_ERR_{name} \(1u << (\d+)\)", hdr)
            assert m and (1 << int(m.group(1))) == getattr(E, f"ERR_{name}")


def test_scalar_bin():                                  # test_ops.py:52-65
    assert H.ScalarBin.of(0.67, 0.01).bin == 33
    assert H.ScalarBin.of(3.14, 0.01).bin == 157
    assert H.ScalarBin.of(-0.67, 0.01).bin == -33
    assert H.ScalarBin.of(0.019, 0.01).bin == 0
    with pytest.raises(H.QuantOverflow):
        H.ScalarBin.of(1e300, 1e-10)


def test_reduction_finalize_matches_reference_expressions():
    from paper_2408_11971_b200 import ops

    rng = np.random.default_rng(5)
    for _ in range(50):
        bins = rng.integers(-(2 ** 40), 2 ** 40, int(rng.integers(1, 500)))
        S = int(bins.astype(object).sum())
        Q = int((bins.astype(object) ** 2).sum())
        eps = float(rng.choice([1e-3, 0.25, 2.0 ** -7]))
        n = bins.size
        assert ops.mean_from(S, n, eps) == O.mean_from(S, n, eps)
        assert ops.variance_from(S, Q, n, eps) == O.variance_from(S, Q, n, eps)
    # 128/192-bit limb round trip
    for S, Q in ((-(2 ** 100) + 7, 2 ** 170 + 3), (5, 0), (-1, 2 ** 64)):
        m = (1 << 64) - 1
        limbs = np.array([S & m, (S >> 64) & m, Q & m, (Q >> 64) & m, (Q >> 128) & m],
                         dtype=np.uint64)
        assert ops.unpack_moments(limbs) == (S, Q)


def test_dispatch_tables_mirror_the_reference():   # ops.py:37-48
    assert H.STREAM_OPS == {"neg": (1, False), "sadd": (1, True), "ssub": (1, True),
                            "smul": (1, True), "eadd": (2, False), "esub": (2, False),
                            "hadamard": (2, False)}
    assert H.REDUCTIONS == {"mean": 1, "variance": 1, "stddev": 1, "covariance": 2, "ssim": 2}
    with pytest.raises(ValueError):
        H.apply_stream_op("neg", [])
