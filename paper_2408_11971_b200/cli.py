"""Command-line front end on the B200 path: the
reference's subcommands, flags, report formats, CSV schema and exit codes
(reference ``cli.py:1-419``), with every operation on the GPU.

    python -m paper_2408_11971_b200.cli compress field.f32 -o f.hsz --dims 100x500x500 \\
        --eps 1e-4 --eps-mode rel
    python -m paper_2408_11971_b200.cli op smul f.hsz -o g.hsz --scalar -1.25 --verify
    python -m paper_2408_11971_b200.cli stats variance g.hsz --verify --report csv
    python -m paper_2408_11971_b200.cli bench --dims 256x256x64 --eps 1e-3 --report csv
    python -m paper_2408_11971_b200.cli distsim --nodes 4 --dims 128x128 --eps 1e-3

``--verify`` runs the traditional workflow -- fully decompress, operate in
the float64 value domain, recompress (reference ``ops.py:559-634``) -- also
on the GPU (torch float64 on the decompressed values + this package's
compressor), and compares like the reference does.  Timings are wall clock
around each call including its synchronisation, like the reference's.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

from . import codec, ops
from .distsim import aggregate_homomorphic
from .errors import HoszpError, VerificationMismatch
from .model import QuantArray, QuantParams, deserialize, serialize

CSV_COLUMNS = ["op", "bytes_in", "cr", "t_homo_s", "t_oracle_s", "speedup", "max_abs_diff"]
CSV_EXTRA_COLUMNS = ["node_count", "eps"]
COMMANDS = ("compress", "decompress", "op", "stats", "bench", "distsim")
EXIT_OK, EXIT_USAGE, EXIT_IO, EXIT_CODEC, EXIT_VERIFY = 0, 2, 3, 4, 5
REDUCTION_RTOL = 1e-9


def _torch():
    import torch

    return torch


# ---------------------------------------------------------------------------
# synthetic fields (reference synth.py:10-27)

def smooth_field(dims, seed: int = 0, dtype: str = "f32") -> codec.RawArray:
    """A few low-frequency cosine waves per axis, deterministic amplitudes
    and phases (the reference's default bench / distsim field)."""
    return codec.RawArray(smooth_values(dims, seed), tuple(int(d) for d in dims), dtype)


def smooth_values(dims, seed: int = 0) -> np.ndarray:
    """The float64 values of smooth_field, flattened."""
    rng = np.random.default_rng(seed)
    dims = tuple(int(d) for d in dims)
    fld = np.zeros(dims, dtype=np.float64)
    for axis, d in enumerate(dims):
        x = np.linspace(0.0, 1.0, d, dtype=np.float64)
        wave = np.zeros(d, dtype=np.float64)
        for freq in (1.0, 2.0, 5.0):
            amp = rng.uniform(0.2, 1.0) / freq
            phase = rng.uniform(0.0, 2.0 * np.pi)
            wave += amp * np.cos(2.0 * np.pi * freq * x + phase)
        shape = [1] * len(dims)
        shape[axis] = d
        fld += wave.reshape(shape)
    return fld.ravel()


# ---------------------------------------------------------------------------
# the traditional workflow on the GPU (reference ops.py:559-634)

def _values64(stream):
    """float64 reconstruction on the device (codec.py:511-513)."""
    ds = codec._as_device_stream(stream)
    return codec.decompress(ds, out_dtype=np.float64).values


def _nearest(v, eps):
    """codec.py:163-171: round-half-away requantization of values."""
    t = _torch()
    q = v / (2.0 * eps)
    mag = t.floor(t.abs(q) + 0.5)
    if bool((mag >= 2.0 ** 63).any()):
        from .errors import QuantOverflow
        raise QuantOverflow("requantized bin exceeds 63-bit range")
    return t.where(q < 0, -mag, mag).to(t.int64)


def _rescale(products, eps):
    """ops.py:199-208 on a device int64 tensor of exact products."""
    t = _torch()
    tt = (2.0 * eps) * products.to(t.float64)
    mag = t.floor(t.abs(tt) + 0.5)
    if bool((mag >= 2.0 ** 63).any()):
        from .errors import QuantOverflow
        raise QuantOverflow("rescaled bin exceeds 63-bit range")
    return t.where(tt < 0, -mag, mag).to(t.int64)


def oracle_stream(name, streams, scalar=None):
    t = _torch()
    p = streams[0].params
    for other in streams[1:]:
        ops._check_params(streams[0], other)
    vals = [_values64(s) for s in streams]
    p64 = QuantParams(p.eps, p.dims, p.block_len, "f64")
    if name in ("smul", "hadamard"):
        ra = _nearest(vals[0], p.eps)
        if name == "smul":
            rb = ops.ScalarBin.of(scalar, p.eps).bin
            ma, mb = int(ra.abs().max().item()) if ra.numel() else 0, abs(rb)
            if ma and mb and ma > (2 ** 63 - 1) // mb:
                raise NotImplementedError("--verify: products beyond int64")
            prod = ra * rb
        else:
            rb = _nearest(vals[1], p.eps)
            ma = int(ra.abs().max().item()) if ra.numel() else 0
            mb = int(rb.abs().max().item()) if rb.numel() else 0
            if ma and mb and ma > (2 ** 63 - 1) // mb:
                raise NotImplementedError("--verify: products beyond int64")
            prod = ra * rb
        return codec.encode_from_quant(QuantArray(_rescale(prod, p.eps), p64))
    if name == "neg":
        out = -vals[0]
    elif name == "sadd":
        out = vals[0] + ops.ScalarBin.of(scalar, p.eps).quantized_value
    elif name == "ssub":
        out = vals[0] - ops.ScalarBin.of(scalar, p.eps).quantized_value
    elif name == "eadd":
        out = vals[0] + vals[1]
    elif name == "esub":
        out = vals[0] - vals[1]
    else:
        raise ValueError(f"unknown stream op {name!r}")
    return codec.compress(codec.RawArray(out.contiguous(), p.dims, "f64"), p64)


def oracle_reduction(name, streams):
    for other in streams[1:]:
        ops._check_params(streams[0], other)
    vals = [_values64(s) for s in streams]
    if name == "mean":
        return float(vals[0].mean())
    if name == "variance":
        return float(vals[0].var(unbiased=False))
    if name == "stddev":
        return float(vals[0].std(unbiased=False))
    va = vals[0]
    vb = vals[1]
    if name == "covariance":
        return float(((va - va.mean()) * (vb - vb.mean())).mean())
    if name == "ssim":
        mu_a, mu_b = float(va.mean()), float(vb.mean())
        var_a, var_b = float(va.var(unbiased=False)), float(vb.var(unbiased=False))
        cov = float(((va - mu_a) * (vb - mu_b)).mean())
        value_range = max(float(va.max() - va.min()), float(vb.max() - vb.min()))
        c1 = (0.01 * value_range) ** 2
        c2 = (0.03 * value_range) ** 2
        den = (mu_a * mu_a + mu_b * mu_b + c1) * (var_a + var_b + c2)
        if den == 0.0:
            raise ValueError("SSIM is undefined: degenerate zero-range operands")
        return float((2.0 * mu_a * mu_b + c1) * (2.0 * cov + c2) / den)
    raise ValueError(f"unknown reduction {name!r}")


def _max_abs_diff(a, b) -> float:
    va, vb = _values64(a), _values64(b)
    return float((va - vb).abs().max()) if va.numel() else 0.0


# ---------------------------------------------------------------------------
# reports (reference cli.py:175-213)

def _emit(rows, fmt, file=None):
    file = file or sys.stdout
    if fmt == "json":
        print(json.dumps(rows, indent=2), file=file)
        return
    if fmt == "csv":
        columns = [c for c in CSV_COLUMNS + CSV_EXTRA_COLUMNS
                   if c in CSV_COLUMNS or any(c in r for r in rows)]
        print(",".join(columns), file=file)
        for row in rows:
            print(",".join(str(row.get(c, "")) for c in columns), file=file)
        return
    for row in rows:
        print("  ".join(f"{c}={v}" for c, v in row.items()), file=file)


def _row(name, t_homo, bytes_in, cr, t_oracle=None, max_abs_diff=None, **extra):
    row = {
        "op": name,
        "bytes_in": bytes_in,
        "cr": f"{cr:.4g}",
        "t_homo_s": f"{t_homo:.6g}",
        "t_oracle_s": "" if t_oracle is None else f"{t_oracle:.6g}",
        "speedup": "" if t_oracle is None else
                   f"{t_oracle / t_homo:.4g}" if t_homo > 0 else "inf",
        "max_abs_diff": "" if max_abs_diff is None else repr(max_abs_diff),
        "throughput_Bps": f"{(bytes_in / t_homo if t_homo > 0 else 0.0):.6g}",
    }
    row.update(extra)
    return row


def _timed(fn):
    t = _torch()
    t.cuda.synchronize()
    t0 = time.perf_counter()
    out = fn()
    t.cuda.synchronize()
    return out, time.perf_counter() - t0


def _load(paths):
    out = []
    for path in paths:
        with open(path, "rb") as fh:
            out.append(codec._as_device_stream(deserialize(fh.read())))
    return out


# ---------------------------------------------------------------------------
# subcommands

def _cmd_compress(a) -> int:
    t = _torch()
    raw = codec.read_raw(a.input, a.dims, a.dtype)
    dev = codec.RawArray(t.from_numpy(raw.numpy()).cuda(), a.dims, a.dtype)
    eps = codec.resolve_eps(dev, a.eps, a.eps_mode)
    params = QuantParams(eps, a.dims, a.block_len, a.dtype)
    s, dt = _timed(lambda: codec.compress(dev, params))
    data = serialize(s.to_host())
    with open(a.output, "wb") as fh:
        fh.write(data)
    _emit([_row("compress", dt, raw.nbytes, raw.nbytes / len(data))], a.report)
    return EXIT_OK


def _cmd_decompress(a) -> int:
    (s,) = _load([a.input])
    out, dt = _timed(lambda: codec.decompress(s))
    codec.write_raw(codec.RawArray(out.values.cpu().numpy(), out.dims, out.dtype), a.output)
    _emit([_row("decompress", dt, s.serialized_size, s.compression_ratio)], a.report)
    return EXIT_OK


def _cmd_op(a) -> int:
    streams = _load(a.inputs)
    arity, needs_scalar = ops.STREAM_OPS[a.op_name]
    if len(streams) != arity:
        print(f"hoszp: {a.op_name} takes {arity} input stream(s)", file=sys.stderr)
        return EXIT_USAGE
    if needs_scalar and a.scalar is None:
        print(f"hoszp: {a.op_name} requires --scalar", file=sys.stderr)
        return EXIT_USAGE
    res, dt = _timed(lambda: ops.apply_stream_op(a.op_name, streams, a.scalar))
    if a.output:
        with open(a.output, "wb") as fh:
            fh.write(serialize(res.to_host()))
    bytes_in = sum(s.params.raw_nbytes for s in streams)
    t_or = diff = None
    if a.verify:
        z, t_or = _timed(lambda: oracle_stream(a.op_name, streams, a.scalar))
        diff = _max_abs_diff(res, z)
    _emit([_row(a.op_name, dt, bytes_in, res.compression_ratio, t_or, diff)], a.report)
    if diff is not None and diff != 0.0:
        print(f"hoszp: error kind=VerificationMismatch: max abs diff {diff}", file=sys.stderr)
        return EXIT_VERIFY
    return EXIT_OK


def _cmd_stats(a) -> int:
    streams = _load(a.inputs)
    if len(streams) != ops.REDUCTIONS[a.op_name]:
        print(f"hoszp: {a.op_name} takes {ops.REDUCTIONS[a.op_name]} input stream(s)",
              file=sys.stderr)
        return EXIT_USAGE
    value, dt = _timed(lambda: ops.apply_reduction(a.op_name, streams))
    print(f"{a.op_name} = {value!r}")
    t_or = diff = want = None
    ok = True
    if a.verify:
        want, t_or = _timed(lambda: oracle_reduction(a.op_name, streams))
        diff = abs(value - want)
        ok = diff <= REDUCTION_RTOL * max(abs(want), abs(value), 1e-300)
    _emit([_row(a.op_name, dt, sum(s.params.raw_nbytes for s in streams),
                streams[0].compression_ratio, t_or, diff)], a.report)
    if not ok:
        print(f"hoszp: error kind=VerificationMismatch: |{value!r} - {want!r}| = {diff}",
              file=sys.stderr)
        return EXIT_VERIFY
    return EXIT_OK


def bench_rows(raw, params, names=None, scalar=3.14):
    """Compress once, then time each operation against the traditional
    workflow (reference cli.py:287-333)."""
    t = _torch()
    dev = codec.RawArray(t.from_numpy(raw.numpy()).cuda(), raw.dims, raw.dtype)
    stream, dt = _timed(lambda: codec.compress(dev, params))
    rows = [_row("compress", dt, raw.nbytes, raw.nbytes / stream.serialized_size)]
    names = names or (list(ops.STREAM_OPS) + list(ops.REDUCTIONS))
    second = None
    for name in names:
        arity = ops.STREAM_OPS[name][0] if name in ops.STREAM_OPS else ops.REDUCTIONS[name]
        operands = [stream]
        if arity == 2:
            if second is None:
                second = ops.scalar_add(stream, 16.0 * params.eps)
            operands = [stream, second]
        if name in ops.STREAM_OPS:
            res, th = _timed(lambda: ops.apply_stream_op(name, operands, scalar))
            z, to = _timed(lambda: oracle_stream(name, operands, scalar))
            diff = _max_abs_diff(res, z)
        else:
            value, th = _timed(lambda: ops.apply_reduction(name, operands))
            want, to = _timed(lambda: oracle_reduction(name, operands))
            diff = abs(value - want)
        rows.append(_row(name, th, sum(s.params.raw_nbytes for s in operands),
                         stream.compression_ratio, to, diff))
    return rows


def _cmd_bench(a) -> int:
    raw = codec.read_raw(a.input, a.dims, a.dtype) if a.input else smooth_field(a.dims, a.seed, a.dtype)
    eps = codec.resolve_eps(raw, a.eps, a.eps_mode)
    params = QuantParams(eps, a.dims, a.block_len, a.dtype)
    names = a.ops_list.split(",") if a.ops_list else None
    unknown = set(names or []) - set(ops.STREAM_OPS) - set(ops.REDUCTIONS)
    if unknown:
        print(f"hoszp: unknown ops {sorted(unknown)}", file=sys.stderr)
        return EXIT_USAGE
    _emit(bench_rows(raw, params, names, a.scalar), a.report)
    return EXIT_OK


def _cmd_distsim(a) -> int:
    """Homomorphic vs traditional sum aggregation of node streams
    (reference distsim.py:113-146)."""
    t = _torch()
    if a.nodes < 2:
        print("hoszp: --nodes must be >= 2", file=sys.stderr)
        return EXIT_USAGE
    if a.input:
        chunk = codec.read_raw(a.input, a.dims, a.dtype)
        arrays = [chunk] * a.nodes
    else:
        arrays = [smooth_field(a.dims, a.seed + i, a.dtype) for i in range(a.nodes)]
    params = QuantParams(a.eps, a.dims, a.block_len, a.dtype)
    streams = [codec.compress(codec.RawArray(t.from_numpy(r.numpy()).cuda(), r.dims, r.dtype), params)
               for r in arrays]
    bytes_c = sum(s.serialized_size for s in streams)
    bytes_in = sum(r.nbytes for r in arrays)
    t_h = t_t = float("inf")
    for _ in range(max(1, a.reps)):
        homo, dt = _timed(lambda: aggregate_homomorphic(streams))
        t_h = min(t_h, dt)

        def trad():
            tot = _values64(streams[0]).clone()
            for s in streams[1:]:
                tot += _values64(s)
            p64 = QuantParams(params.eps, params.dims, params.block_len, "f64")
            return codec.compress(codec.RawArray(tot, params.dims, "f64"), p64)

        trd, dt = _timed(trad)
        t_t = min(t_t, dt)
    diff = _max_abs_diff(homo, trd)
    if diff != 0.0:
        raise VerificationMismatch("homomorphic and traditional aggregates decompress "
                                   f"differently (max abs diff {diff})")
    _emit([_row("distsim_sum", t_h, bytes_in, bytes_in / bytes_c, t_t, diff,
                node_count=a.nodes, eps=a.eps)], a.report)
    return EXIT_OK


# ---------------------------------------------------------------------------
# parser (reference cli.py:113-171)

def _parse_dims(text):
    try:
        dims = tuple(int(part) for part in text.lower().split("x"))
    except ValueError:
        raise argparse.ArgumentTypeError(f"bad dims {text!r}, expected e.g. 500x500x100")
    if not dims or any(d < 1 for d in dims):
        raise argparse.ArgumentTypeError(f"dims must be positive, got {text!r}")
    return dims


def build_parser():
    ap = argparse.ArgumentParser(prog="hoszp-b200", description="HoSZp on B200")
    sub = ap.add_subparsers(dest="command", required=True)

    def common(p):
        p.add_argument("--threads", type=int, default=None, help="accepted and ignored (GPU)")
        p.add_argument("--report", choices=["text", "csv", "json"], default="text")

    p = sub.add_parser("compress")
    p.add_argument("input")
    p.add_argument("-o", "--output", required=True)
    p.add_argument("--dims", type=_parse_dims, required=True)
    p.add_argument("--dtype", choices=["f32", "f64"], default="f32")
    p.add_argument("--eps", type=float, required=True)
    p.add_argument("--eps-mode", choices=["abs", "rel"], default="abs")
    p.add_argument("--block-len", type=int, default=32)
    common(p)
    p = sub.add_parser("decompress")
    p.add_argument("input")
    p.add_argument("-o", "--output", required=True)
    common(p)
    p = sub.add_parser("op")
    p.add_argument("op_name", metavar="name", choices=sorted(ops.STREAM_OPS))
    p.add_argument("inputs", nargs="+")
    p.add_argument("-o", "--output")
    p.add_argument("--scalar", type=float)
    p.add_argument("--verify", action="store_true")
    common(p)
    p = sub.add_parser("stats")
    p.add_argument("op_name", metavar="name", choices=sorted(ops.REDUCTIONS))
    p.add_argument("inputs", nargs="+")
    p.add_argument("--verify", action="store_true")
    common(p)
    p = sub.add_parser("bench")
    p.add_argument("--input")
    p.add_argument("--dims", type=_parse_dims, required=True)
    p.add_argument("--dtype", choices=["f32", "f64"], default="f32")
    p.add_argument("--eps", type=float, required=True)
    p.add_argument("--eps-mode", choices=["abs", "rel"], default="abs")
    p.add_argument("--block-len", type=int, default=32)
    p.add_argument("--ops", dest="ops_list", default=None)
    p.add_argument("--scalar", type=float, default=3.14)
    p.add_argument("--seed", type=int, default=0)
    common(p)
    p = sub.add_parser("distsim")
    p.add_argument("--nodes", type=int, default=4)
    p.add_argument("--dims", type=_parse_dims, required=True)
    p.add_argument("--dtype", choices=["f32", "f64"], default="f32")
    p.add_argument("--eps", type=float, required=True)
    p.add_argument("--block-len", type=int, default=32)
    p.add_argument("--input")
    p.add_argument("--reps", type=int, default=3)
    p.add_argument("--latency-per-byte", type=float, default=0.0)
    p.add_argument("--seed", type=int, default=0)
    common(p)
    return ap


_COMMANDS = {"compress": _cmd_compress, "decompress": _cmd_decompress, "op": _cmd_op,
             "stats": _cmd_stats, "bench": _cmd_bench, "distsim": _cmd_distsim}


def main(argv=None) -> int:
    args = build_parser().parse_args(argv)
    if getattr(args, "eps", None) is not None and not args.eps > 0:
        print("hoszp: error kind=ValueError: eps must be positive", file=sys.stderr)
        return EXIT_USAGE
    try:
        return _COMMANDS[args.command](args)
    except VerificationMismatch as exc:
        print(f"hoszp: error kind=VerificationMismatch: {exc}", file=sys.stderr)
        return EXIT_VERIFY
    except HoszpError as exc:
        print(f"hoszp: error kind={type(exc).__name__}: {exc}", file=sys.stderr)
        return EXIT_CODEC
    except OSError as exc:
        print(f"hoszp: error kind=IOError: {exc}", file=sys.stderr)
        return EXIT_IO
    except ValueError as exc:
        print(f"hoszp: error kind=ValueError: {exc}", file=sys.stderr)
        return EXIT_USAGE


if __name__ == "__main__":
    os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
    sys.exit(main())
