"""Config 5 as ONE field (2048^3 float32, 2^33 values, 32 GiB) on the GPU:
single-GPU stream vs the same field split over 2, 3 and 4 ranks.

north_star: the field is partitioned by contiguous block ranges; compress
takes the relative eps from the GLOBAL value range (C1, codec.py:96-99),
the shards' sections concatenated at the C2 offsets are the single-field
stream (blocks are independent and byte-aligned, pkg/FORMAT.md:39-40), and
mean / variance come from the exact partial sums (C3, ops.py:360-393).

* The parent (this pytest process) runs the whole chain on the whole field
  on cuda:0: value range -> compress -> negate -> scalar_add 3.5 ->
  scalar_mul -1.25 -> exact S, Q -> decompress.  It keeps the compressed and
  the chained stream's sections on the device and a per-block checksum of
  the decompressed values.
* World sizes 2, 3, 4: spawned ranks (gloo, all on cuda:0 -- their kernels
  never wait on each other; only the host collectives do) generate exactly
  their block range of the same field (``workloads.config5_range``), run C1,
  the chain with the CUDA kernels, C2 and C3 (sharding.Collectives), and
  compare their sections BYTE FOR BYTE against the parent's device sections
  at the C2 offsets (the parent's tensors arrive over CUDA IPC), their S/Q and
  mean/variance bit-for-bit, their decompressed values by per-block
  checksums.
* Oracle parity: a block-aligned 2^27-value slice straddling the slab 3 / 4
  boundary (the 2-rank shard boundary) is compressed and chained by the CPU
  oracle at the GLOBAL eps and compared with the same block range of the
  parent's streams and decompressed values.
"""

import os
import socket
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu

N_FIELD = 1 << 33
SADD, SMUL = 3.5, -1.25
SLICE = (1 << 32) - (1 << 26), (1 << 32) + (1 << 26)      # 2^27 values across slabs 3 | 4


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def block_checksums(values, e0):
    """Per-block checksum of float32 values whose first element is global
    element e0 (block aligned): sum_i bits(v_i) * c(i) mod 2^64 with c(i) a
    64-bit mix of the GLOBAL element index -- equal sums for equal blocks,
    position-sensitive, computed in chunks on the device."""
    import torch

    assert e0 % 32 == 0
    n = values.numel()
    out = torch.empty(-(-n // 32), dtype=torch.int64, device=values.device)
    step = 1 << 27
    for a in range(0, n, step):
        b = min(n, a + step)
        v = values[a:b].view(torch.int32).to(torch.int64)
        i = torch.arange(e0 + a, e0 + b, dtype=torch.int64, device=values.device)
        c = (i * -7046029254386353131) ^ (i >> 17)        # wraps mod 2^64
        c = c * 6364136223846793005 + 1442695040888963407
        prod = v * c
        m = prod.numel()
        full = m // 32 * 32
        out[a // 32:a // 32 + m // 32] = prod[:full].view(-1, 32).sum(1)
        if full < m:
            out[a // 32 + m // 32] = prod[full:].sum()
        del v, i, c, prod
    return out


def _sections(ds):
    sb, pb = ds.totals()
    return (ds.widths, ds.outliers, ds.signs[:sb], ds.payload[:pb])


@pytest.fixture(scope="module")
def single():
    """The whole field on one GPU (parent process)."""
    import torch

    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    sys.path.insert(0, ROOT)
    import paper_2408_11971_b200 as H
    from paper_2408_11971_b200 import ops
    from paper_2408_11971_b200 import workloads as W

    torch.cuda.set_device(0)
    rel = W.CONFIGS[5]["rel_eps"]
    x = W.config5_range(0, N_FIELD)
    raw = H.RawArray(x, (2048, 2048, 2048), "f32")
    lo, hi = raw.value_range()
    eps = rel * (hi - lo)
    p = H.QuantParams(eps, (2048, 2048, 2048), 32, "f32")
    s = H.compress(raw, p)
    xs_host = x[SLICE[0]:SLICE[1]].cpu().numpy()
    del raw, x
    torch.cuda.empty_cache()
    z = H.scalar_mul(H.scalar_add(H.negate(s), SADD), SMUL)
    S, Q = ops.exact_moments(z, want_sq=True)
    vals = H.decompress(z).values
    csum = block_checksums(vals, 0)
    slice_vals = vals[SLICE[0]:SLICE[1]].cpu().numpy()
    del vals
    torch.cuda.empty_cache()
    s.check()
    yield dict(H=H, eps=eps, lo=lo, hi=hi, s=s, z=z, S=S, Q=Q, csum=csum,
               xs=xs_host, slice_vals=slice_vals)
    del s, z, csum
    torch.cuda.empty_cache()


def _rank_worker(rank, world, port, refs, want, outdir, host_shm):
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist

    torch.cuda.set_device(0)
    import paper_2408_11971_b200 as H
    from paper_2408_11971_b200 import ops
    from paper_2408_11971_b200 import workloads as W
    from paper_2408_11971_b200.sharding import Collectives, element_range

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import datetime
    import faulthandler

    faulthandler.dump_traceback_later(900, exit=True)       # a hung rank shows where it hangs
    dist.init_process_group("gloo", rank=rank, world_size=world,
                            timeout=datetime.timedelta(seconds=300))
    msgs = []
    try:
        coll = Collectives(host_shm=host_shm)
        e0, e1 = element_range(N_FIELD, 32, rank, world)
        b0 = e0 // 32
        # one rank at a time generates its range: the slab FFTs' scratch is
        # then never needed by several processes at once on the shared GPU
        x = None
        for r in range(world):
            if r == rank:
                x = W.config5_range(e0, e1)
                torch.cuda.synchronize()
                torch.cuda.empty_cache()
            coll.barrier()
        n = e1 - e0
        raw = H.RawArray(x, (n,), "f32")
        lo, hi = coll.global_range(*raw.value_range())                     # C1
        eps = W.CONFIGS[5]["rel_eps"] * (hi - lo)
        if (lo, hi, eps) != (want["lo"], want["hi"], want["eps"]):
            msgs.append(f"C1: range/eps {(lo, hi, eps)} != {(want['lo'], want['hi'], want['eps'])}")
        p = H.QuantParams(eps, (n,), 32, "f32")
        s = H.compress(raw, p)
        del raw, x
        torch.cuda.empty_cache()
        z = H.scalar_mul(H.scalar_add(H.negate(s), SADD), SMUL)
        lay_s, lay_z = coll.global_offsets_many(b0, [s.totals(), z.totals()])     # C2
        for name, mine, lay, ref in (("compress", s, lay_s, refs["s"]), ("chain", z, lay_z, refs["z"])):
            w, o, sg, py = _sections(mine)
            rw, ro, rsg, rpy = ref
            if (lay.sign_total, lay.payload_total) != (rsg.numel(), rpy.numel()):
                msgs.append(f"{name}: C2 totals {(lay.sign_total, lay.payload_total)} != "
                            f"{(rsg.numel(), rpy.numel())}")
                continue
            checks = (("widths", w, rw[b0:b0 + w.numel()]),
                      ("outliers", o, ro[b0:b0 + o.numel()]),
                      ("signs", sg, rsg[lay.sign_offset:lay.sign_offset + sg.numel()]),
                      ("payload", py, rpy[lay.payload_offset:lay.payload_offset + py.numel()]))
            for sec, a, b in checks:
                if a.numel() != b.numel() or not torch.equal(a, b):
                    msgs.append(f"{name}: section {sec} differs from the single-GPU stream at "
                                f"the C2 offsets (rank {rank}/{world})")
        S, _ = ops.exact_moments(z, want_sq=False)
        S1, _ = coll.global_moments(S, 0)                                    # C3 (mean)
        S2, Q = ops.exact_moments(z, want_sq=True)
        S2, Q2 = coll.global_moments(S2, Q)                                  # C3 (variance)
        if (S1, S2, Q2) != (want["S"], want["S"], want["Q"]):
            msgs.append(f"C3: moments {(S1, Q2)} != {(want['S'], want['Q'])}")
        if ops.mean_from(S1, N_FIELD, eps) != want["mean"] or \
                ops.variance_from(S2, Q2, N_FIELD, eps) != want["var"]:
            msgs.append("mean / variance differ from the single-GPU values")
        vals = H.decompress(z).values
        cs = block_checksums(vals, e0)
        if not torch.equal(cs, refs["csum"][b0:b0 + cs.numel()]):
            bad = int((cs != refs["csum"][b0:b0 + cs.numel()]).sum().item())
            msgs.append(f"decompress: {bad} blocks differ (rank {rank}/{world})")
        z.check()
    except Exception as e:          # reported through the file: every rank reaches the barrier
        msgs.append(f"rank {rank}: {type(e).__name__}: {e}")
    finally:
        with open(os.path.join(outdir, f"rank{rank}.txt"), "w") as f:
            f.write("\n".join(msgs) if msgs else "ok")
        dist.destroy_process_group()


@pytest.mark.parametrize("world,host_shm", [(2, False), (3, True), (4, False)])
def test_config5_sharded_equals_single_gpu(single, tmp_path, world, host_shm):
    import torch.multiprocessing as mp

    from paper_2408_11971_b200 import ops

    d = single
    refs = {"s": _sections(d["s"]), "z": _sections(d["z"]), "csum": d["csum"]}
    eps = d["eps"]
    want = {"lo": d["lo"], "hi": d["hi"], "eps": eps, "S": d["S"], "Q": d["Q"],
            "mean": ops.mean_from(d["S"], N_FIELD, eps),
            "var": ops.variance_from(d["S"], d["Q"], N_FIELD, eps)}
    mp.spawn(_rank_worker, args=(world, _free_port(), refs, want, str(tmp_path), host_shm),
             nprocs=world, join=True)
    got = [(tmp_path / f"rank{r}.txt").read_text() for r in range(world)]
    assert all(g == "ok" for g in got), "\n".join(got)


def test_config5_slice_vs_oracle_at_global_eps(single):
    """A block-aligned 2^27-value slice of the whole-field streams equals the
    oracle's compress / chain / decompress of that slice at the global eps."""
    import torch

    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import hoszp_oracle as O

    d = single
    e0, e1 = SLICE
    b0, b1 = e0 // 32, e1 // 32
    m = e1 - e0

    def block_range_of(ds):
        w = ds.widths[:b1].to(torch.int64)
        # every block before the slice is a full 32-value block: 4 sign bytes
        # if non-constant, 4 w payload bytes
        so = int((4 * (w[:b0] > 0)).sum().item())
        po = int((4 * w[:b0]).sum().item())
        sl = int((4 * (w[b0:] > 0)).sum().item())
        pl = int((4 * w[b0:]).sum().item())
        return (ds.widths[b0:b1].cpu().numpy(), ds.outliers[b0:b1].cpu().numpy(),
                ds.signs[so:so + sl].cpu().numpy().tobytes(),
                ds.payload[po:po + pl].cpu().numpy().tobytes())

    ref = O.compress(d["xs"], d["eps"], (m,), 32, "f32")
    w, o, sg, py = block_range_of(d["s"])
    assert w.tobytes() == ref["widths"].tobytes()
    assert np.array_equal(o, ref["outliers"])
    assert sg == ref["signs"] and py == ref["payload"]
    zr = O.scalar_mul(O.scalar_add(O.negate(ref), SADD), SMUL)
    w, o, sg, py = block_range_of(d["z"])
    assert w.tobytes() == zr["widths"].tobytes()
    assert np.array_equal(o, zr["outliers"])
    assert sg == zr["signs"] and py == zr["payload"]
    assert d["slice_vals"].tobytes() == O.decompress(zr).tobytes()
