"""The GPU-backed CLI: the reference's subcommands,
CSV schema and exit codes, with --verify running the traditional workflow
on the GPU.  Streams written by the CLI are checked against the oracle."""

import numpy as np
import pytest

import hoszp_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cli():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2408_11971_b200 import cli as mod

    return mod


def test_compress_op_stats_pipeline(cli, tmp_path, capsys):
    n = 64 * 1000 + 3
    i = np.arange(n)
    x = (np.sin(i / 333.0) * 20 + 5 + np.cos(i / 71.0)).astype(np.float32)
    raw = tmp_path / "x.f32"
    x.tofile(raw)
    f = tmp_path / "x.hsz"
    assert cli.main(["compress", str(raw), "-o", str(f), "--dims", str(n), "--eps", "1e-3",
                     "--eps-mode", "rel", "--report", "csv"]) == 0
    out = capsys.readouterr().out.splitlines()
    assert out[0] == ",".join(cli.CSV_COLUMNS)
    eps = O.resolve_eps(x, 1e-3, "rel")
    assert f.read_bytes() == O.serialize(O.compress(x, eps, (n,), 32, "f32"))
    g = tmp_path / "g.hsz"
    for args in (["op", "smul", str(f), "-o", str(g), "--scalar", "-1.25", "--verify"],
                 ["op", "neg", str(f), "--verify"], ["op", "eadd", str(f), str(f), "--verify"],
                 ["op", "hadamard", str(f), str(f), "--verify"],
                 ["stats", "variance", str(f), "--verify"], ["stats", "ssim", str(f), str(f), "--verify"],
                 ["stats", "mean", str(f), "--verify", "--report", "json"]):
        assert cli.main(args) == 0, args
    want = O.scalar_mul(O.compress(x, eps, (n,), 32, "f32"), -1.25)
    assert g.read_bytes() == O.serialize(want)
    d = tmp_path / "g.f32"
    assert cli.main(["decompress", str(g), "-o", str(d)]) == 0
    assert d.read_bytes() == O.decompress(want).tobytes()


def test_bench_and_distsim(cli, capsys):
    assert cli.main(["bench", "--dims", "64x48x20", "--eps", "1e-3", "--eps-mode", "rel",
                     "--report", "csv"]) == 0
    rows = capsys.readouterr().out.strip().splitlines()
    assert rows[0].split(",") == cli.CSV_COLUMNS
    names = [r.split(",")[0] for r in rows[1:]]
    assert names[0] == "compress" and "hadamard" in names and "ssim" in names
    assert cli.main(["distsim", "--nodes", "3", "--dims", "96x40", "--eps", "1e-3",
                     "--reps", "1", "--report", "csv"]) == 0
    rows = capsys.readouterr().out.strip().splitlines()
    assert rows[0].split(",")[-2:] == ["node_count", "eps"]


def test_exit_codes(cli, tmp_path):
    assert cli.main(["op", "sadd", str(tmp_path / "missing.hsz"), "--scalar", "1"]) == cli.EXIT_IO
    bad = tmp_path / "bad.hsz"
    bad.write_bytes(b"XSZP" + bytes(40))
    assert cli.main(["stats", "mean", str(bad)]) == cli.EXIT_CODEC
    assert cli.main(["distsim", "--nodes", "1", "--dims", "8", "--eps", "0.1"]) == cli.EXIT_USAGE
