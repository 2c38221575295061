"""Device-side stream assembly and .hsz file I/O:
serialize_device / write_hsz / read_hsz against the reference's bytes
(golden fixtures) and the reference's error classes for malformed files."""

import numpy as np
import pytest

from conftest import load_golden

pytestmark = pytest.mark.gpu

CASES = [c for c in load_golden() if c.has("stream")]


@pytest.fixture(scope="module")
def H():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2408_11971_b200 as mod

    return mod


@pytest.mark.parametrize("case", CASES[::4], ids=repr)
def test_read_write_round_trip(H, tmp_path, case):
    from paper_2408_11971_b200 import hszio

    data = case.bytes_of("stream")
    path = tmp_path / "s.hsz"
    path.write_bytes(data)
    ds = hszio.read_hsz(str(path))
    assert H.serialize(ds.to_host()) == data
    assert hszio.serialize_device(ds).cpu().numpy().tobytes() == data
    out = tmp_path / "t.hsz"
    assert hszio.write_hsz(ds, str(out), chunk=4096) == len(data)
    assert out.read_bytes() == data
    assert np.array_equal(H.decode_to_quant(ds).bins.cpu().numpy(), case["bins_out"])


def test_large_device_stream(H, tmp_path):
    import torch

    from paper_2408_11971_b200 import hszio

    n = 1 << 22
    x = torch.sin(torch.arange(n, device="cuda", dtype=torch.float32) / 999.0) * 50 + 7
    raw = H.RawArray(x, (n,), "f32")
    p = H.QuantParams(H.resolve_eps(raw, 1e-4, "rel"), (n,), 32, "f32")
    s = H.compress(raw, p)
    want = H.serialize(s.to_host())
    path = str(tmp_path / "big.hsz")
    assert hszio.write_hsz(s, path, chunk=1 << 20) == len(want)
    assert open(path, "rb").read() == want
    back = hszio.read_hsz(path, chunk=1 << 20)
    assert H.decompress(back).values.cpu().numpy().tobytes() == \
        H.decompress(s).values.cpu().numpy().tobytes()


def test_malformed_files_raise_reference_errors(H, tmp_path):
    from paper_2408_11971_b200 import hszio

    data = next(c for c in CASES if len(c.bytes_of("stream")) > 200).bytes_of("stream")
    bad = {
        "magic": b"XSZP" + data[4:],
        "version": data[:4] + bytes([9]) + data[5:],
        "short": data[:10],
        "dims": data[:21],
        "widths": data[:len(data) // 4],
        "payload": data[:-1],
        "trailing": data + b"\0",
    }
    for name, blob in bad.items():
        path = tmp_path / f"{name}.hsz"
        path.write_bytes(blob)
        with pytest.raises(Exception) as want:
            H.deserialize(blob)
        with pytest.raises(Exception) as got:
            hszio.read_hsz(str(path))
        assert type(got.value) is type(want.value), name
