"""allreduce_streams on the GPU path: device-resident streams, the
reduce-scatter over tile-aligned block ranges, the on-device fold of each
rank's range (headroom branch and the pairwise elementwise_add branch) and
the reassembly -- checked byte for byte against the oracle's single-process
fold.  The ranks share cuda:0 and exchange over gloo (the collectives move
compressed bytes; no kernel of one rank waits on another's)."""

import os
import socket
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu

CASES = {
    # name: (n, eps)
    "fields": (32 * 128 * 7 + 13, 0.004),
    "wide": (32 * 128 * 2 + 5, 0.5),       # widths 63: no int64 headroom, pairwise fold
}


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _operand(case, n, eps, r):
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import hoszp_oracle as O

    rng = np.random.default_rng(100 + r)
    if case == "wide":
        # +-A alternating (residuals ~2A: width 63), sign flipped per rank so
        # the sums stay inside int64
        A = 3 << 60
        i = np.arange(n)
        bins = np.where(i % 2 == 0, A, -A).astype(np.int64) * (1 if r % 2 == 0 else -1)
        bins += rng.integers(-1000, 1000, n, dtype=np.int64)
        bins[::32] = rng.integers(-1000, 1000, bins[::32].size)
        return O.encode_bins(bins, eps, (n,), 32, "f32")
    i = np.arange(n)
    x = (np.sin(i / (300 + 40 * r)) * 20 + rng.normal(0, 0.05, n)).astype(np.float32)
    return O.compress(x, eps, (n,), 32, "f32")


def _worker(rank, world, port, outdir, case):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import torch
    import torch.distributed as dist

    import hoszp_oracle as O
    import paper_2408_11971_b200 as H
    from paper_2408_11971_b200.device import DeviceStream
    from paper_2408_11971_b200.sharding import Collectives

    torch.cuda.set_device(0)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import datetime
    import faulthandler

    faulthandler.dump_traceback_later(300, exit=True)       # a hung rank shows where it hangs
    dist.init_process_group("gloo", rank=rank, world_size=world,
                            timeout=datetime.timedelta(seconds=240))
    try:
        coll = Collectives()
        n, eps = CASES[case]
        mine = DeviceStream.from_host(H.deserialize(O.serialize(_operand(case, n, eps, rank))))
        got = coll.allreduce_streams(mine)
        assert isinstance(got, DeviceStream)
        blob = H.serialize(got.to_host())
        # the device stream is usable as is (tile-offset cache rebuilt)
        m = H.mean(got)
        parts = [None] * world
        dist.all_gather_object(parts, (blob, m))
        if rank == 0:
            np.save(os.path.join(outdir, "agg.npy"), np.array(parts, dtype=object),
                    allow_pickle=True)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,case", [(2, "fields"), (3, "fields"), (2, "wide"), (3, "wide")])
def test_allreduce_streams_device(tmp_path, world, case):
    import torch

    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import torch.multiprocessing as mp

    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import hoszp_oracle as O

    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path), case), nprocs=world, join=True)
    parts = list(np.load(tmp_path / "agg.npy", allow_pickle=True))
    n, eps = CASES[case]
    ops = [_operand(case, n, eps, r) for r in range(world)]
    if case == "wide":
        assert not O._headroom(ops)
    want = O.aggregate_homomorphic(ops)
    ws = O.serialize(want)
    S, _ = O.moments(want)
    for blob, m in parts:
        assert blob == ws
        assert m == O.mean_from(S, n, eps)


def _nccl_worker(rank, world, port, outdir):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import torch
    import torch.distributed as dist

    import hoszp_oracle as O
    import paper_2408_11971_b200 as H
    from paper_2408_11971_b200.device import DeviceStream
    from paper_2408_11971_b200.sharding import Collectives

    torch.cuda.set_device(0)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("nccl", rank=rank, world_size=world)
    try:
        coll = Collectives()
        assert coll.device.type == "cuda"
        n, eps = CASES["fields"]
        mine = DeviceStream.from_host(H.deserialize(O.serialize(_operand("fields", n, eps, 0))))
        got = coll.allreduce_streams(mine)
        with open(os.path.join(outdir, "nccl.bin"), "wb") as f:
            f.write(H.serialize(got.to_host()))
    finally:
        dist.destroy_process_group()


def test_allreduce_streams_nccl_single_rank(tmp_path):
    """The NCCL code path (device-resident send/receive buffers, no host
    staging) at world size 1: the aggregate of one stream is the stream."""
    import torch

    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import torch.multiprocessing as mp

    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import hoszp_oracle as O

    mp.spawn(_nccl_worker, args=(1, _free_port(), str(tmp_path)), nprocs=1, join=True)
    n, eps = CASES["fields"]
    assert (tmp_path / "nccl.bin").read_bytes() == O.serialize(_operand("fields", n, eps, 0))
