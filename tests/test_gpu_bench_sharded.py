"""bench.py's multi-rank mode measures the north_star split: ONE config-5
field (2048^3) partitioned by contiguous block ranges, C1 global eps, C2
global section offsets, C3 exact moments.  Run it at N = 1 and under
torchrun at N = 2 (both ranks on cuda:0, collectives on gloo -- the pool has
one GPU per box) and require identical digests of the WHOLE compressed
stream, the WHOLE chained stream (sections at their C2 offsets) and the
decompressed field, and bit-identical eps / mean / variance."""

import json
import os
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _line(out):
    lines = [ln for ln in out.splitlines() if ln.startswith("{")]
    assert lines, out[-2000:]
    return json.loads(lines[-1])


def test_config5_two_ranks_equal_one():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    args = ["bench.py", "--config", "5", "--quick", "--steps", "1", "--warmup", "1"]
    env = dict(os.environ)
    one = subprocess.run([sys.executable] + args, cwd=ROOT, env=env, capture_output=True,
                         text=True, timeout=900)
    assert one.returncode == 0, one.stderr[-3000:]
    d1 = _line(one.stdout)
    env2 = dict(env, HSZ_DIST_BACKEND="gloo")
    two = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                          "--nproc-per-node", "2", "--master-addr", "127.0.0.1",
                          "--master-port", str(_free_port())] + args + ["--gpus", "2"],
                         cwd=ROOT, env=env2, capture_output=True, text=True, timeout=1200)
    assert two.returncode == 0, two.stderr[-3000:]
    d2 = _line(two.stdout)
    assert d1["n_gpus"] == 1 and d2["n_gpus"] == 2
    assert d1["config"]["global_elements"] == d2["config"]["global_elements"] == 1 << 33
    assert d2["config"]["elements_per_gpu"] == 1 << 32
    assert d1["digests"] == d2["digests"]


def test_config5_nccl_collectives_world1():
    """The NCCL code paths of C1-C3 (device tensors, all_reduce MIN /
    all_gather / all_reduce SUM on a real NCCL communicator) under torchrun
    with one rank: same digests as the plain single-GPU run (the pool has
    one GPU per box, so this is the NCCL world this machine can form)."""
    import torch

    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    args = ["bench.py", "--config", "5", "--quick", "--steps", "1", "--warmup", "1"]
    one = subprocess.run([sys.executable] + args, cwd=ROOT, capture_output=True, text=True,
                         timeout=900)
    assert one.returncode == 0, one.stderr[-3000:]
    env = dict(os.environ, HSZ_FORCE_COLL="1")
    nccl = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                           "--nproc-per-node", "1", "--master-addr", "127.0.0.1",
                           "--master-port", str(_free_port())] + args,
                          cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert nccl.returncode == 0, nccl.stderr[-3000:]
    d1, dn = _line(one.stdout), _line(nccl.stdout)
    assert "nccl" in dn["config"]["parallelism"]
    assert d1["digests"] == dn["digests"]

