"""Latency of the chain's small collectives (C1 value range, C2 offsets, C3
moments) per call, on the process group torchrun sets up:

    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 \
        tools/coll_latency.py
"""
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2408_11971_b200.sharding import Collectives  # noqa: E402


def t_of(fn, reps=200):
    for _ in range(20):
        fn()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return round(1e6 * statistics.median(ts), 1)


local = int(os.environ.get("LOCAL_RANK", "0"))
torch.cuda.set_device(local)
dist.init_process_group(os.environ.get("HSZ_DIST_BACKEND", "nccl"),
                        device_id=torch.device("cuda", local))
out = {}
for name, kw in (("torch.distributed", {"host_shm": False}), ("host shm", {"host_shm": True})):
    coll = Collectives(**kw)
    out[name] = {
        "global_range_us": t_of(lambda: coll.global_range(1.0, 2.0)),
        "global_offsets_us": t_of(lambda: coll.global_offsets(0, 1000, 2000)),
        "global_moments_us": t_of(lambda: coll.global_moments(-12345, 678910)),
        "global_moments_offsets_us": t_of(
            lambda: coll.global_moments_offsets(-12345, 678910, 0, [(1, 2), (3, 4)])),
        "max_over_ranks_us": t_of(lambda: coll.max_over_ranks(1.5)),
    }
if dist.get_rank() == 0:
    import json

    print(json.dumps({"world": dist.get_world_size(), **out}))
dist.destroy_process_group()
