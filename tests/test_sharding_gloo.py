"""Multi-rank path on CPU (gloo, world_size 2 and 3): contiguous block-range
sharding + the three collectives (C1 global range, C2 global section
offsets, C3 exact moments).  The per-shard codec here is the CPU oracle (the
GPU kernels are covered by the -m gpu suite); what is under test is the
partitioning and collective logic of paper_2408_11971_b200/sharding.py:
the concatenated shards must equal the single-process stream byte for byte,
and mean / variance must be bit-identical for any rank count."""

import os
import socket
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


import datetime  # noqa: E402

_PG_TIMEOUT = datetime.timedelta(seconds=180)   # a stuck peer fails the test, not the suite


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _field(n, seed=3):
    rng = np.random.default_rng(seed)
    return (np.cumsum(rng.normal(0, 0.3, n)) + 280).astype(np.float32)


def _worker(rank, world, port, n, rel, outdir, host_shm=True):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import torch.distributed as dist

    import hoszp_oracle as O
    from paper_2408_11971_b200.sharding import Collectives, element_range

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world, timeout=_PG_TIMEOUT)
    try:
        coll = Collectives(host_shm=host_shm)
        assert coll.host_shm == host_shm
        x = _field(n)
        k = 32
        e0, e1 = element_range(n, k, rank, world)
        xs = x[e0:e1]
        lo, hi = coll.global_range(float(xs.min()), float(xs.max()))     # C1
        eps = float(rel) * (hi - lo)
        s = O.compress(xs, eps, (xs.size,), k, "f32")
        lay = coll.global_offsets(e0 // k, len(s["signs"]), len(s["payload"]))   # C2
        S, Q = O.moments(s)
        St, Qt = coll.global_moments(S, Q)                                # C3
        assert coll.max_over_ranks(float(rank) + 0.5) == world - 0.5
        S2, Q2, lays = coll.global_moments_offsets(S, Q, e0 // k,
                                                   [(len(s["signs"]), len(s["payload"])), (3, 5)])
        assert (S2, Q2) == (St, Qt) and lays[0] == lay
        assert (lays[1].sign_offset, lays[1].payload_total) == (3 * rank, 5 * world)
        assert coll.global_offsets_many(e0 // k, [(len(s["signs"]), len(s["payload"])),
                                                  (3, 5)]) == lays
        parts = [None] * world
        dist.all_gather_object(parts, (lay.__dict__, s["widths"].tobytes(),
                                       np.asarray(s["outliers"], np.int64).tobytes(),
                                       s["signs"], s["payload"], St, Qt, eps))
        if rank == 0:
            np.save(os.path.join(outdir, "parts.npy"), np.array(parts, dtype=object),
                    allow_pickle=True)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,host_shm", [(2, True), (3, True), (2, False), (3, False)])
def test_sharded_equals_single_process(tmp_path, world, host_shm):
    """C1-C3 over the node-local shared-memory exchange and over the process
    group give the single-process stream, eps and moments."""
    import torch.multiprocessing as mp

    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import hoszp_oracle as O
    from paper_2408_11971_b200 import sharding

    n, rel = 32 * 997 + 13, 1e-4
    mp.spawn(_worker, args=(world, _free_port(), n, rel, str(tmp_path), host_shm), nprocs=world,
             join=True)
    parts = list(np.load(tmp_path / "parts.npy", allow_pickle=True))
    x = _field(n)
    eps = O.resolve_eps(x, rel, "rel")
    ref = O.compress(x, eps, (n,), 32, "f32")
    assert all(p[7] == eps for p in parts)                       # C1: identical eps everywhere
    widths = b"".join(p[1] for p in parts)
    outl = np.concatenate([np.frombuffer(p[2], np.int64) for p in parts])
    signs = b"".join(p[3] for p in parts)
    payload = b"".join(p[4] for p in parts)
    assert widths == ref["widths"].tobytes()
    assert np.array_equal(outl, ref["outliers"])
    assert signs == ref["signs"] and payload == ref["payload"]
    # C2 offsets are the prefix sums of the shard sections
    acc_s = acc_p = 0
    for p in parts:
        lay = p[0]
        assert lay["sign_offset"] == acc_s and lay["payload_offset"] == acc_p
        assert lay["sign_total"] == len(ref["signs"]) and lay["payload_total"] == len(ref["payload"])
        acc_s += len(p[3])
        acc_p += len(p[4])
    # C3: exact global moments -> bit-identical mean / variance
    S, Q = O.moments(ref)
    assert all((p[5], p[6]) == (S, Q) for p in parts)
    assert O.mean_from(parts[0][5], n, eps) == O.mean(ref)
    assert O.variance_from(parts[0][5], parts[0][6], n, eps) == O.variance(ref)


def test_block_ranges_partition_exactly():
    from paper_2408_11971_b200.sharding import block_range, element_range

    for nb in (1, 7, 128, 1000, 781250):
        for world in (1, 2, 3, 4, 8):
            spans = [block_range(nb, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == nb
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1
    # every shard boundary is block aligned; the tail block is the last shard's
    n = 32 * 10 + 5
    ranges = [element_range(n, 32, r, 3) for r in range(3)]
    assert all(a % 32 == 0 for a, _ in ranges) and ranges[-1][1] == n


def test_tile_block_ranges_partition_exactly():
    from paper_2408_11971_b200.sharding import tile_block_range

    for nb in (1, 127, 128, 129, 128 * 7 + 3, 100_000):
        for world in (1, 2, 3, 5, 8):
            rs = [tile_block_range(nb, r, world) for r in range(world)]
            assert rs[0][0] == 0 and rs[-1][1] == nb
            assert all(rs[i][1] == rs[i + 1][0] for i in range(world - 1))
            assert all((b0 % 128 == 0 or b0 == nb) and b0 <= b1 for b0, b1 in rs)


def test_limb_packing_round_trip():
    from paper_2408_11971_b200.sharding import _from_limbs, _to_limbs

    for S, Q in ((0, 0), (-5, 7), (-(2 ** 120), 2 ** 191 - 1), (2 ** 126, 2 ** 64)):
        assert _from_limbs(_to_limbs(S, Q)) == (S, Q)


STREAM_CASES = {
    # name: (n, per-rank field seeds offset, eps)
    "ragged": (32 * 300 + 7, 10, 0.01),
    "multi_tile": (32 * 128 * 5 + 19, 20, 0.002),
    "one_tile": (32 * 50, 30, 0.01),          # fewer tiles than ranks: empty ranges
}


def _stream_worker(rank, world, port, outdir, case):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import torch.distributed as dist

    import hoszp_oracle as O
    import paper_2408_11971_b200 as H
    from paper_2408_11971_b200.sharding import Collectives

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world, timeout=_PG_TIMEOUT)
    try:
        coll = Collectives()
        n, seed, eps = STREAM_CASES[case]
        x = _field(n, seed=seed + rank)
        mine = H.deserialize(O.serialize(O.compress(x, eps, (n,), 32, "f32")))

        def oracle_fold(streams):
            agg = O.aggregate_homomorphic([O.deserialize(H.serialize(s)) for s in streams])
            return H.deserialize(O.serialize(agg))

        got = coll.allreduce_streams(mine, fold=oracle_fold)
        parts = [None] * world
        dist.all_gather_object(parts, H.serialize(got))
        if rank == 0:
            np.save(os.path.join(outdir, "agg.npy"), np.array(parts, dtype=object), allow_pickle=True)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,case", [(2, "ragged"), (3, "ragged"), (2, "multi_tile"),
                                        (3, "multi_tile"), (3, "one_tile")])
def test_allreduce_streams(tmp_path, world, case):
    """Reduce-scatter over tile-aligned block ranges + all-gather of the
    partial sums: every rank ends with the single-process fold's stream,
    byte for byte (slices folded by the oracle, reassembled here)."""
    import torch.multiprocessing as mp

    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import hoszp_oracle as O

    mp.spawn(_stream_worker, args=(world, _free_port(), str(tmp_path), case), nprocs=world,
             join=True)
    parts = list(np.load(tmp_path / "agg.npy", allow_pickle=True))
    n, seed, eps = STREAM_CASES[case]
    streams = [O.compress(_field(n, seed=seed + r), eps, (n,), 32, "f32") for r in range(world)]
    want = O.serialize(O.aggregate_homomorphic(streams))
    assert all(p == want for p in parts)


def _err_worker(rank, world, port, outdir):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import torch.distributed as dist

    import paper_2408_11971_b200 as H
    from paper_2408_11971_b200.sharding import Collectives

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world, timeout=_PG_TIMEOUT)
    try:
        coll = Collectives()
        n = 32 * 128 * 3
        p = H.QuantParams(0.5, (n,), 32, "f32")
        mine = H.CompressedStream(p, np.zeros(n // 32, np.uint8), np.full(n // 32, 7, np.int32),
                                  b"", b"")

        def failing_fold(streams):
            # only the rank owning the last tile fails; all ranks must raise
            if coll.rank == world - 1:
                raise H.OutlierOverflow("outlier out of signed 32-bit range")
            return streams[0]

        try:
            coll.allreduce_streams(mine, fold=failing_fold)
            outcome = "none"
        except H.OutlierOverflow:
            outcome = "OutlierOverflow"
        q = H.QuantParams(0.25 if rank == 1 else 0.5, (n,), 32, "f32")
        other = H.CompressedStream(q, mine.widths, mine.outliers, b"", b"")
        try:
            coll.allreduce_streams(other)
            mismatch = "none"
        except H.ParamsMismatch:
            mismatch = "ParamsMismatch"
        parts = [None] * world
        dist.all_gather_object(parts, (outcome, mismatch))
        if rank == 0:
            np.save(os.path.join(outdir, "err.npy"), np.array(parts, dtype=object), allow_pickle=True)
    finally:
        dist.destroy_process_group()


def test_allreduce_streams_errors_agree(tmp_path):
    """A fold error on one rank is raised on every rank (same class); params
    differing across ranks raise ParamsMismatch everywhere (ops.py:77-81)."""
    import torch.multiprocessing as mp

    mp.spawn(_err_worker, args=(3, _free_port(), str(tmp_path)), nprocs=3, join=True)
    parts = list(np.load(tmp_path / "err.npy", allow_pickle=True))
    assert all(tuple(p) == ("OutlierOverflow", "ParamsMismatch") for p in parts)


def _write_worker(rank, world, port, path):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import torch.distributed as dist

    import hoszp_oracle as O
    import paper_2408_11971_b200 as H
    from paper_2408_11971_b200.sharding import Collectives, element_range

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world, timeout=_PG_TIMEOUT)
    try:
        coll = Collectives()
        n, k = 32 * 700 + 9, 32
        x = _field(n, seed=5)
        e0, e1 = element_range(n, k, rank, world)
        xs = x[e0:e1]
        lo, hi = coll.global_range(float(xs.min()), float(xs.max()))
        eps = 1e-4 * (hi - lo)
        shard = H.deserialize(O.serialize(O.compress(xs, eps, (xs.size,), k, "f32")))
        lay = coll.global_offsets(e0 // k, len(shard.sign_planes), len(shard.payload))
        coll.write_sharded(path, H.QuantParams(eps, (n,), k, "f32"), lay, shard)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_write_sharded_equals_serialize(tmp_path, world):
    """Per-rank pwrites at the C2 offsets produce exactly the single-process
    .hsz bytes (FORMAT.md) of the whole field."""
    import torch.multiprocessing as mp

    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import hoszp_oracle as O

    path = str(tmp_path / "field.hsz")
    mp.spawn(_write_worker, args=(world, _free_port(), path), nprocs=world, join=True)
    n = 32 * 700 + 9
    x = _field(n, seed=5)
    eps = 1e-4 * (float(x.max()) - float(x.min()))
    want = O.serialize(O.compress(x, eps, (n,), 32, "f32"))
    assert open(path, "rb").read() == want


def _hc_worker(rank, world, port, outdir):
    sys.path.insert(0, ROOT)
    import torch.distributed as dist

    from paper_2408_11971_b200.sharding import HostAllGather

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world, timeout=_PG_TIMEOUT)
    try:
        hc = HostAllGather(dist, None, rank, world, timeout_s=60)
        rows = []
        for r in range(300):                       # many rounds: the double buffer is reused
            nv = 1 + (r % HostAllGather.MAX_VALS)
            vals = [rank * 1_000_003 + r * 7 + j - (1 << 62) for j in range(nv)]
            got = hc(vals)
            want = [[q * 1_000_003 + r * 7 + j - (1 << 62) for j in range(nv)]
                    for q in range(world)]
            rows.append(got == want)
        with open(os.path.join(outdir, f"hc{rank}.txt"), "w") as f:
            f.write("ok" if all(rows) else "mismatch")
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_host_allgather_rounds(tmp_path, world):
    """The shared-memory all-gather: 300 back-to-back rounds of 1..40 words,
    every rank sees every rank's words of the same round."""
    import torch.multiprocessing as mp

    mp.spawn(_hc_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    assert all((tmp_path / f"hc{r}.txt").read_text() == "ok" for r in range(world))


def test_chunk_packing_sums_exactly():
    """C3 on the process group: ten 32-bit chunks per rank, one allreduce SUM,
    exact recombination -- also when S is negative on some ranks and the
    totals carry across chunks."""
    from paper_2408_11971_b200.sharding import _from_chunks, _to_chunks

    cases = [(0, 0), (-5, 7), (-(2 ** 120), 2 ** 191 - 1), (2 ** 126 - 1, 2 ** 64), (-1, 1)]
    for S, Q in cases:
        assert _from_chunks(_to_chunks(S, Q)) == (S, Q)
    ranks = [(-(2 ** 100) + 3, 2 ** 150 + 9), (2 ** 99, 2 ** 150 - 1), (-7, 0), (5, 2 ** 40)]
    summed = [sum(col) for col in zip(*(_to_chunks(S, Q) for S, Q in ranks))]
    assert _from_chunks(summed) == (sum(S for S, _ in ranks), sum(Q for _, Q in ranks))


def _shm_fail_worker(rank, world, port, outdir, fail_rank):
    sys.path.insert(0, ROOT)
    import torch.distributed as dist

    from paper_2408_11971_b200 import sharding

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world, timeout=_PG_TIMEOUT)
    try:
        if rank == fail_rank:
            # this rank cannot see the segment (a private IPC namespace)
            real_open = os.open

            def no_shm(path, *a, **k):
                if "hsz_coll_" in str(path):
                    raise FileNotFoundError(path)
                return real_open(path, *a, **k)

            os.open = no_shm
        coll = sharding.Collectives(host_shm=True)
        lo, hi = coll.global_range(float(rank), float(rank) + 1.0)
        S, Q = coll.global_moments(-rank - 1, 2 ** 70 + rank)
        lay = coll.global_offsets(rank, 10 + rank, 100 + rank)
        with open(os.path.join(outdir, f"shm{rank}.txt"), "w") as f:
            f.write(repr((coll.host_shm, lo, hi, S, Q, lay.sign_offset, lay.payload_total)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,fail_rank", [(2, 1), (3, 0), (3, 2)])
def test_host_shm_setup_failure_falls_back_on_every_rank(tmp_path, world, fail_rank):
    """A rank that cannot map the shared-memory segment (same hostname, other
    IPC namespace) makes EVERY rank fall back to the process group together
    -- no rank blocks in a barrier while another crashes."""
    import torch.multiprocessing as mp

    mp.spawn(_shm_fail_worker, args=(world, _free_port(), str(tmp_path), fail_rank),
             nprocs=world, join=True)
    got = [eval((tmp_path / f"shm{r}.txt").read_text()) for r in range(world)]
    S = sum(-r - 1 for r in range(world))
    Q = sum(2 ** 70 + r for r in range(world))
    tot_s = sum(10 + r for r in range(world))
    tot_p = sum(100 + r for r in range(world))
    for r, g in enumerate(got):
        assert g[0] is False
        assert g[1:5] == (0.0, float(world), S, Q)
        assert g[5] == sum(10 + q for q in range(r)) and g[6] == tot_p
    assert tot_s > 0
