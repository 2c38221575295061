"""CLI plumbing that needs no GPU: the parser mirrors the reference's
subcommands and flags (reference cli.py:113-171), the CSV schema and the
usage exit codes."""

import pytest

from paper_2408_11971_b200 import cli


def test_commands_and_schema():
    assert cli.COMMANDS == ("compress", "decompress", "op", "stats", "bench", "distsim")
    assert cli.CSV_COLUMNS == ["op", "bytes_in", "cr", "t_homo_s", "t_oracle_s", "speedup",
                               "max_abs_diff"]
    assert (cli.EXIT_OK, cli.EXIT_USAGE, cli.EXIT_IO, cli.EXIT_CODEC, cli.EXIT_VERIFY) == \
        (0, 2, 3, 4, 5)


def test_parser_accepts_reference_invocations():
    p = cli.build_parser()
    a = p.parse_args(["compress", "x.f32", "-o", "x.hsz", "--dims", "100x500x500", "--eps", "1e-4",
                      "--eps-mode", "rel", "--block-len", "32", "--threads", "8", "--report", "csv"])
    assert a.dims == (100, 500, 500) and a.eps_mode == "rel" and a.report == "csv"
    a = p.parse_args(["op", "smul", "a.hsz", "-o", "b.hsz", "--scalar", "-1.25", "--verify"])
    assert a.op_name == "smul" and a.verify and a.scalar == -1.25
    a = p.parse_args(["stats", "ssim", "a.hsz", "b.hsz"])
    assert a.inputs == ["a.hsz", "b.hsz"]
    a = p.parse_args(["distsim", "--nodes", "4", "--dims", "64x64", "--eps", "1e-3"])
    assert a.nodes == 4
    for name in ("neg", "sadd", "ssub", "smul", "eadd", "esub", "hadamard"):
        p.parse_args(["op", name, "a.hsz"])
    for name in ("mean", "variance", "stddev", "covariance", "ssim"):
        p.parse_args(["stats", name, "a.hsz"])


@pytest.mark.parametrize("argv", [["compress", "x", "-o", "y", "--dims", "0x3", "--eps", "1"],
                                  ["compress", "x", "-o", "y", "--dims", "ax3", "--eps", "1"],
                                  ["op", "nope", "a.hsz"]])
def test_usage_errors(argv):
    with pytest.raises(SystemExit) as e:
        cli.main(argv)
    assert e.value.code == cli.EXIT_USAGE


def test_nonpositive_eps_is_usage_error():
    assert cli.main(["compress", "x", "-o", "y", "--dims", "4", "--eps", "-1"]) == cli.EXIT_USAGE


def test_smooth_field_is_deterministic():
    a = cli.smooth_values((16, 8), seed=3)
    b = cli.smooth_values((16, 8), seed=3)
    assert a.shape == (128,) and (a == b).all() and not (a == cli.smooth_values((16, 8), 4)).all()
