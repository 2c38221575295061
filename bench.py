"""Benchmark of the HoSZp hot path on B200 (one JSON line on rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 2|4|5]
    python bench.py --impl reference ...       # CPU arm (rank 0 only)

Workload.  Every config is ONE field partitioned by contiguous block ranges
across the ranks (north_star; rank r owns ``sharding.element_range(N, 32, r,
world)``), so ``scaling`` is "strong" and ``value`` covers the whole field:

* default at N = 1: **config 4** -- the 512^3 float32 lognormal field
  (exp(1.5 G), G a Gaussian random field with P(k) ~ k^-2, seed 3), relative
  error bound 1e-3, block_len 32: the largest BASELINE.json config pinned to
  one GPU; 512 MiB of input, 4x the 126 MB L2.  The field is generated ONCE on
  the host (numpy, ``workloads.config4``) and the same values feed both arms.
* default at N > 1: **config 5** -- the 2048^3 field (2^33 values, 32 GiB),
  generated per slab from (seed 4, slab) on each rank's GPU
  (``workloads.config5_range``), so the field is identical for any N.  C1
  (global value range -> the one relative eps), C2 (allgather of the shard
  byte counts -> global section offsets) and C3 (allreduce of the exact
  moment partial sums) run on NCCL.  The N = 1 line carries the same
  config-5 chain on one GPU under ``config5_n1`` (the scaling baseline).

One step is the whole op chain of the path on the field:

    value range (K0) -> C1 -> resolve rel eps -> compress (K1) -> negate (K4)
    -> scalar_add (K5) -> scalar_mul (K6) -> mean (K7) + C3
    -> variance (K7) + C3 -> decompress (K3) [+ C2]

``value`` = 7 ops x 4N uncompressed bytes of the whole field / device step
time (max over ranks).  Inputs are resident in HBM; L2 is flushed with a
512 MB read between steps (excluded from the timing).  ``e2e`` runs the same
chain through the public API from the field in pinned HOST memory (H2D
inside the timed region) and ends with a D2H of the resulting stream
sections and the decompressed field.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

OPS = ("compress", "negate", "scalar_add", "scalar_mul", "mean", "variance", "decompress")
METRIC = "uncompressed GB/s per op (compress/decompress/homomorphic) & % HBM roofline"
L2_BYTES = 126 << 20


def _traffic(config, op):
    """DRAM bytes per launch of `op`'s kernel (dram__bytes_read.sum +
    dram__bytes_write.sum) from the committed ncu --set full capture of this
    config (profiles/traffic.json), if any."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            v = json.load(f).get(f"config{config}", {}).get(op)
        return int(v) if v is not None else None
    except Exception:
        return None


def _issue(config, op):
    """Issue-side numbers of `op`'s kernel from the committed ncu --set full
    capture of this config (profiles/issue.json): thread-instructions per
    element, issue-slot utilisation, IPC -- the ceiling this block format
    actually runs into (tools/ncu_issue.py)."""
    try:
        with open(os.path.join(ROOT, "profiles", "issue.json")) as f:
            v = json.load(f).get(f"config{config}", {}).get(op)
        return {k: v[k] for k in ("thread_inst_per_element", "issue_slots_busy_pct", "ipc")} \
            if v else None
    except Exception:
        return None


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            m = json.load(f)
        return float(m["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# ---------------------------------------------------------------------------
# clocks sampled during the timed region (nvidia-smi, like the recipe)

class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
            t0 = time.time()
            while not self.lines and time.time() - t0 < 5.0:   # wait for the first sample
                time.sleep(0.02)
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], [], set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# the workload: one field, a contiguous block range per rank

def _default_config(world: int) -> int:
    return 4 if world == 1 else 5


def _global_dims(config: int):
    from paper_2408_11971_b200 import workloads as W

    return tuple(W.CONFIGS[config]["dims"])


def _count(dims) -> int:
    n = 1
    for d in dims:
        n *= int(d)
    return n


_HOST_FIELDS = {}


def host_field(config: int):
    """The host (numpy float32) field of configs 1-4 -- generated once per
    process; both arms use exactly these values."""
    from paper_2408_11971_b200 import workloads as W

    if config not in _HOST_FIELDS:
        _HOST_FIELDS[config] = W.field(config)
    return _HOST_FIELDS[config]


def shard_field(config: int, rank: int, world: int, device):
    """(x on `device`, e0, e1): this rank's elements [e0, e1) of the field."""
    import torch

    from paper_2408_11971_b200 import workloads as W
    from paper_2408_11971_b200.sharding import element_range

    n = _count(_global_dims(config))
    e0, e1 = element_range(n, 32, rank, world)
    if config == 5:
        x = W.config5_range(e0, e1, device=device)
    else:
        x = torch.from_numpy(host_field(config)[e0:e1]).to(device)
    return x.contiguous(), e0, e1


class Chain:
    """One step of the op chain on this rank's shard through the public
    (device) API, with the collectives C1-C3 when the field is sharded."""

    def __init__(self, H, cfg, coll, dims_local, n_global, block0):
        self.H = H
        self.cfg = cfg
        self.coll = coll
        self.dims = dims_local
        self.n_global = n_global
        self.block0 = block0
        self.layouts = None      # C2 of the last step (multi-rank)

    def run(self, x, events=None, host_out=False):
        H, cfg = self.H, self.cfg
        # events: {mark index: CUDA event}; only the given marks are recorded
        # (the timed steps record 0 and 7 only: each record is host time that
        # would otherwise sit between a synchronising call and the next launch)
        mark = (lambda i: events[i].record() if i in events else None) if events is not None \
            else (lambda i: None)
        mark(0)
        raw = H.RawArray(x, self.dims, "f32")                  # K0: range + finite check
        lo, hi = raw.value_range()
        if self.coll is not None:
            lo, hi = self.coll.global_range(lo, hi)            # C1
        eps = float(cfg["rel_eps"]) * (hi - lo)
        p = H.QuantParams(eps, self.dims, 32, "f32")
        s = H.compress(raw, p)                                 # K1
        if self.coll is not None:
            s.prefetch_totals()        # C2 inputs: copied back asynchronously
        mark(1)
        z = H.negate(s)                                        # K4
        mark(2)
        z = H.scalar_add(z, cfg["sadd"])                       # K5
        mark(3)
        z = H.scalar_mul(z, cfg["smul"])                       # K6
        if self.coll is not None:
            z.prefetch_totals()
        mark(4)
        mean = global_mean(z, self.coll, self.n_global)        # K7 (+ C3)
        mark(5)
        var = global_variance(z, self.coll, self.n_global)     # K7 (+ C3)
        mark(6)
        out = H.decompress(z)                                  # K3
        if self.coll is not None:
            # C2 for the compressed field and the result while decompress runs
            # (their totals were prefetched; nothing in the step waits on it)
            self.layouts = self.coll.global_offsets_many(self.block0, [s.totals(), z.totals()])
        mark(7)
        if host_out:
            from paper_2408_11971_b200.device import download

            hz = z.to_host()
            vals = download([out.values])[0]
            return hz, vals, mean, var
        return z, out, mean, var


def global_mean(z, coll, n_global):
    """ops.mean over the whole field: exact local S, C3, the reference's
    float expression with the GLOBAL element count (ops.py:360-363)."""
    from paper_2408_11971_b200 import ops

    S, Q = ops.exact_moments(z, want_sq=False)
    if coll is not None:
        S, Q = coll.global_moments(S, 0)
    return ops.mean_from(S, n_global, z.params.eps)


def global_variance(z, coll, n_global):
    """ops.variance over the whole field (ops.py:382-393)."""
    from paper_2408_11971_b200 import ops

    S, Q = ops.exact_moments(z, want_sq=True)
    if coll is not None:
        S, Q = coll.global_moments(S, Q)
    return ops.variance_from(S, Q, n_global, z.params.eps)


_MIX_A, _MIX_B, _MIX_C = -7046029254386353131, 6364136223846793005, 1442695040888963407


def _digest(t, off0):
    """Position-weighted checksum of a device tensor's BYTES whose first byte
    sits at global byte offset `off0` of its section: sum_i byte_i * c(off0 + i)
    mod 2^64, c a 64-bit mix of the position.  Shards' digests of the same
    section ADD UP to the whole stream's digest, so the C2-assembled stream
    of N ranks can be compared with the single-GPU stream without gathering
    it (bench.py --digest; tests/test_gpu_bench_sharded.py)."""
    import torch

    u = t.reshape(-1).view(torch.uint8)
    total = torch.zeros((), dtype=torch.int64, device=u.device)
    step = 1 << 26
    for a in range(0, u.numel(), step):
        v = u[a:a + step].to(torch.int64)
        i = torch.arange(off0 + a, off0 + a + v.numel(), dtype=torch.int64, device=u.device)
        c = (i * _MIX_A) ^ (i >> 17)
        c = c * _MIX_B + _MIX_C
        total += (v * c).sum()
        del v, i, c
    return int(total.item()) & ((1 << 64) - 1)


def stream_digests(ds, lay, block0):
    """Digests of the four sections of this rank's shard of a stream at its
    global offsets (C2 layout `lay`; None at N = 1)."""
    sb, pb = ds.totals()
    so = lay.sign_offset if lay is not None else 0
    po = lay.payload_offset if lay is not None else 0
    return [_digest(ds.widths, block0), _digest(ds.outliers, 4 * block0),
            _digest(ds.signs[:sb], so), _digest(ds.payload[:pb], po)]


def chain_digests(H, chain, x, coll):
    """One untimed chain step, then digests of the compressed stream, the
    chained stream and the decompressed values over the WHOLE field (summed
    over ranks), with eps and mean / variance as float hex -- identical for
    any rank count when the sharded path is right."""
    z, out, mean, var = chain.run(x)
    raw = H.RawArray(x, chain.dims, "f32")
    lo, hi = raw.value_range()
    if coll is not None:
        lo, hi = coll.global_range(lo, hi)
    eps = float(chain.cfg["rel_eps"]) * (hi - lo)
    s = H.compress(raw, H.QuantParams(eps, chain.dims, 32, "f32"))
    b0 = chain.block0
    ls = lz = None
    if coll is not None:
        ls, lz = coll.global_offsets_many(b0, [s.totals(), z.totals()])
    vals = [_digest(out.values, 4 * 32 * b0)] + stream_digests(s, ls, b0) + stream_digests(z, lz, b0)
    if coll is not None:
        rows = coll._allgather_i64([v - (1 << 64) if v >= (1 << 63) else v for v in vals])
        vals = [sum(int(r[j]) & ((1 << 64) - 1) for r in rows) & ((1 << 64) - 1)
                for j in range(len(vals))]
    hx = [f"{v:016x}" for v in vals]
    return {"eps": float(eps).hex(), "mean": float(mean).hex(), "variance": float(var).hex(),
            "decompress": hx[0], "compress": hx[1:5], "chain": hx[5:9]}


def _algorithmic_bytes(H, chain, x):
    """Per-op algorithmic bytes of this rank's shard, from
    device-side section totals (no host copy of the streams)."""
    raw = H.RawArray(x, chain.dims, "f32")
    lo, hi = raw.value_range()
    if chain.coll is not None:
        lo, hi = chain.coll.global_range(lo, hi)
    eps = float(chain.cfg["rel_eps"]) * (hi - lo)
    p = H.QuantParams(eps, chain.dims, 32, "f32")
    s = H.compress(raw, p)
    z = H.scalar_mul(H.scalar_add(H.negate(s), chain.cfg["sadd"]), chain.cfg["smul"])
    n = p.element_count
    B = p.block_count
    ss, sp = s.totals()
    zs, zp = z.totals()
    C_in = B + 4 * B + ss + sp
    C_z = B + 4 * B + zs + zp
    nc = int((s.widths > 0).sum().item())
    return {
        "minmax": 4 * n,
        "compress": 4 * n + C_in,
        "negate": 2 * (4 * nc + 4 * B),
        "scalar_add": 2 * 4 * B,
        "scalar_mul": C_in + C_z,
        "mean": C_z,
        "variance": C_z,
        "decompress": C_z + 4 * n,
        "_C": C_in, "_C_chain": C_z,
        "_ratio": p.raw_nbytes / (C_in + 20 + 8 * len(chain.dims)),
        "_eps": eps,
    }


def _flush(flush):
    """Evict L2 with a 512 MB read (clean lines: no write-back charged to the
    next kernel)."""
    flush.view(__import__("torch").int64).max()


def _kernel_times(H, chain, x, flush, reps=10):
    """Mean device time (ms) of each op launched alone after an L2 flush, on
    the stream the op is launched on (torch's current stream: every op of
    the package launches there).  A ~0.2 ms spin kernel is queued first so
    the host enqueues the op while the GPU is busy: the event interval holds
    device time only, not Python launch latency."""
    import torch
    from paper_2408_11971_b200 import _native as N
    from paper_2408_11971_b200 import ops as O
    from paper_2408_11971_b200.device import ptr

    cfg = chain.cfg
    raw = H.RawArray(x, chain.dims, "f32")
    lo, hi = raw.value_range()
    if chain.coll is not None:
        lo, hi = chain.coll.global_range(lo, hi)
    p = H.QuantParams(float(cfg["rel_eps"]) * (hi - lo), chain.dims, 32, "f32")
    s = H.compress(raw, p)
    z0 = H.scalar_add(H.negate(s), cfg["sadd"])
    z = H.scalar_mul(z0, cfg["smul"])
    ctx = s.ctx
    wsp, wsb = ctx.workspace(1, 1)
    mm = ctx.empty(2, torch.float64)
    fns = {
        "minmax": lambda: N.check(ctx.lib.hsz_minmax(ptr(x), N.HSZ_F32, x.numel(), ptr(mm), ctx.err_ptr,
                                                     wsp, wsb, ctx.handle), "hsz_minmax"),
        "compress": lambda: H.compress(raw, p),
        "negate": lambda: H.negate(s),
        "scalar_add": lambda: H.scalar_add(s, cfg["sadd"]),
        "scalar_mul": lambda: H.scalar_mul(z0, cfg["smul"]),
        "mean": lambda: O.moments_device(z, False),
        "variance": lambda: O.moments_device(z, True),
        "decompress": lambda: H.decompress(z),
    }
    out = {}
    for name, fn in fns.items():
        ts = []
        for _ in range(reps + 2):
            _flush(flush)
            torch.cuda._sleep(400_000)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            r = fn()
            b.record()
            torch.cuda.synchronize()
            del r
            ts.append(a.elapsed_time(b))
        out[name] = sum(ts[2:]) / len(ts[2:])
    z.check()
    return out


def _dist_init():
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # HSZ_DIST_BACKEND=gloo: functional check of the N > 1 path with several
    # ranks sharing one GPU (collectives on the host); the default is NCCL
    backend = os.environ.get("HSZ_DIST_BACKEND", "nccl")
    if backend != "nccl":
        local = local % max(1, torch.cuda.device_count())
    # HSZ_FORCE_COLL=1 (under torchrun): the collective path even at N = 1
    if (world > 1 or os.environ.get("HSZ_FORCE_COLL")) and not dist.is_initialized():
        torch.cuda.set_device(local)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    return world, rank, local


def measure(args, config, world, rank, local, coll, light=False):
    """Bench one config on this rank's shard; returns the JSON line (rank 0's
    view, with maxima over ranks).  `light`: chain value and per-op in-chain
    times only (the config-5 scaling baseline at N = 1)."""
    import torch

    import paper_2408_11971_b200 as H
    from paper_2408_11971_b200 import workloads as W

    dev = torch.device("cuda", local)
    cfg = dict(W.CONFIGS[config])
    gdims = _global_dims(config)
    n_global = _count(gdims)
    x, e0, e1 = shard_field(config, rank, world, dev)
    n = x.numel()
    dims_local = gdims if world == 1 else (n,)
    chain = Chain(H, cfg, coll, dims_local, n_global, e0 // 32)
    abytes = _algorithmic_bytes(H, chain, x)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)   # > 126 MB L2

    steps = args.steps if not light else max(3, min(args.steps, 5))
    for _ in range(max(args.warmup, 3) if not (light or args.quick) else max(1, min(args.warmup, 2))):
        chain.run(x)
    torch.cuda.synchronize()

    per_step = []
    if coll is not None:
        coll.barrier()
    torch.cuda.synchronize()
    wall0 = time.perf_counter()
    for _ in range(steps):
        _flush(flush)                                   # evict L2 (excluded from timing)
        evs = {0: torch.cuda.Event(enable_timing=True), 7: torch.cuda.Event(enable_timing=True)}
        chain.run(x, evs)
        torch.cuda.synchronize()
        per_step.append(evs[0].elapsed_time(evs[7]))
    torch.cuda.synchronize()
    if coll is not None:
        coll.barrier()
    wall = time.perf_counter() - wall0
    # per-op breakdown inside the chain: separate (untimed) steps with a mark
    # between every op
    per_op = {op: [] for op in OPS}
    for _ in range(min(steps, 5)):
        _flush(flush)
        evs = {i: torch.cuda.Event(enable_timing=True) for i in range(8)}
        chain.run(x, evs)
        torch.cuda.synchronize()
        for i, op in enumerate(OPS):
            per_op[op].append(evs[i].elapsed_time(evs[i + 1]))

    step_ms = sum(per_step) / len(per_step)
    if coll is not None:
        step_ms = coll.max_over_ranks(step_ms)
    # whole job: 7 ops over the whole field's N elements
    value = len(OPS) * 4.0 * n_global / (step_ms * 1e-3) / 1e9
    field_bytes = 4 * n
    l2_note = (f"per-rank input {field_bytes / 1e6:.0f} MB "
               f"{'>' if field_bytes > L2_BYTES else '<'} 126 MB L2; 512 MB read between "
               f"steps, excluded from timing")
    line = {
        "metric": METRIC,
        "value": round(value, 3),
        "unit": "GB/s",
        "n_gpus": world,
        "steps": steps,
        "warmup": args.warmup,
        "ms_per_step": round(step_ms, 4),
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f64 quantize / int64 bins (f32 input)",
        "data": "synthetic (seeded stand-in for SDRBench; see DESIGN.md)",
        "config": {
            "workload": f"config {config}: {'x'.join(map(str, gdims))} f32, rel eps "
                        f"{cfg['rel_eps']}, block_len 32, op chain {'>'.join(OPS)}, "
                        f"scalars sadd {cfg['sadd']} smul {cfg['smul']}",
            "global_elements": n_global,
            "elements_per_gpu": n,
            "eps": abytes["_eps"],
            "compression_ratio": round(abytes["_ratio"], 3),
            "stream_bytes": int(abytes["_C"]),
            "value_definition": "7 ops x 4N bytes of the whole field / device step time "
                                "(max over ranks)",
            "l2": l2_note,
            "parallelism": (f"{world} ranks, one field by contiguous block ranges, "
                            f"C1/C2/C3 on {coll.backend}"
                            f"{' (host shm for the scalars)' if coll.host_shm else ''}")
            if coll is not None else "1 GPU",
            "wall_s_timed_region": round(wall, 3),
        },
        "ops_in_chain_ms": {op: round(statistics.median(per_op[op]), 4) for op in OPS},
        "gpu_launches": 8 * steps,
    }
    if args.digest or args.quick:
        line["digests"] = chain_digests(H, chain, x, coll)
    if light or args.quick:
        del x, flush
        return line

    # ---- per-kernel timing (each op alone, L2 flushed first) for the roofline
    kern = _kernel_times(H, chain, x, flush, reps=max(10, min(args.steps, 30)))
    peak, peak_kind = _peaks()
    ops_json = {}
    for op in OPS:
        t_ms = statistics.median(per_op[op])
        ops_json[op] = {
            "ms_in_chain": round(t_ms, 4),
            "gbps_uncompressed_in_chain": round(4.0 * n / (t_ms * 1e-3) / 1e9, 2),
            "kernel_ms": round(kern[op], 4),
            "kernel_gbps_uncompressed": round(4.0 * n / (kern[op] * 1e-3) / 1e9, 2),
            "algorithmic_bytes": int(abytes[op]),
            "roofline_frac": round(abytes[op] / (kern[op] * 1e-3) / 1e9 / peak, 4),
            "ncu_issue": _issue(config, op),
        }
    ops_json["minmax"] = {"kernel_ms": round(kern["minmax"], 4),
                          "algorithmic_bytes": int(abytes["minmax"]),
                          "roofline_frac": round(abytes["minmax"] / (kern["minmax"] * 1e-3) / 1e9 / peak, 4)}
    dom = max(OPS, key=lambda o: kern[o])
    achieved = abytes[dom] / (kern[dom] * 1e-3) / 1e9
    traffic = _traffic(config, dom)
    line["ops"] = ops_json
    line["roofline"] = {"bound": "hbm", "kernel": dom, "achieved": round(achieved, 1),
                        "peak": peak, "peak_kind": peak_kind, "unit": "GB/s",
                        "frac": round(achieved / peak, 4),
                        "traffic": traffic,
                        "traffic_source": f"profiles/traffic.json config{config} (ncu --set full)"
                        if traffic is not None else None,
                        "algorithmic_bytes": int(abytes[dom]),
                        "issue": _issue(config, dom)}
    del abytes

    # ---- e2e through the public API from pinned host memory
    if config == 5:
        win = min(n, 1 << 27)
        e2e = _e2e(H, chain, x[:win], flush, steps=max(6, min(args.steps, 12)), coll=coll,
                   dims=(win,), n_global=win * world)
        e2e["window"] = (f"first {win} values of each rank's shard (a 2^27-value window per "
                         f"rank: the whole 2^33-value field does not fit pinned host memory)")
    else:
        e2e = _e2e(H, chain, x, flush, steps=max(6, min(args.steps, 20)), coll=coll,
                   dims=chain.dims, n_global=n_global)
    line["e2e"] = e2e
    del x, flush
    return line


def run_b200(args):
    import torch

    world, rank, local = _dist_init()
    torch.cuda.set_device(local)
    from paper_2408_11971_b200.sharding import Collectives

    coll = Collectives() if world > 1 or os.environ.get("HSZ_FORCE_COLL") else None
    config = args.config or _default_config(world)

    sampler = ClockSampler(local)
    sampler.start()                       # samples cover warm-up, timed steps and kernel timing
    line = measure(args, config, world, rank, local, coll)
    line["clocks"] = sampler.stop()
    if rank == 0 and world == 1 and not args.no_cpu_baseline and config != 5 and not args.quick:
        line["cpu_baseline"] = _cpu_baseline(host_field(config), W_cfg(config),
                                             budget_s=args.cpu_budget)
    if world == 1 and config == 4 and not args.no_scale_baseline and not args.quick:
        # the north_star scaling config on ONE GPU: the baseline of the N > 1 lines
        import gc

        gc.collect()
        torch.cuda.empty_cache()
        try:
            sub = measure(args, 5, world, rank, local, coll, light=True)
            line["config5_n1"] = {k: sub[k] for k in ("value", "unit", "ms_per_step", "steps",
                                                      "config", "ops_in_chain_ms")}
        except torch.cuda.OutOfMemoryError as e:      # report, never fail the headline line
            line["config5_n1"] = {"skipped": f"out of memory: {str(e).splitlines()[0]}"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if coll is not None:
        coll.barrier()
        import torch.distributed as dist

        dist.destroy_process_group()


def W_cfg(config):
    from paper_2408_11971_b200 import workloads as W

    return dict(W.CONFIGS[config])


def _e2e(H, chain, x, flush, steps, coll, dims, n_global):
    """The chain end to end from a pinned HOST field: every step copies the
    field host->device, runs the public API chain and copies the step's
    results (the final stream's four sections, the decompressed field) back
    into a pinned host arena; mean / variance arrive as Python floats."""
    import torch
    from paper_2408_11971_b200.device import download_into

    chain = Chain(H, chain.cfg, chain.coll, dims, n_global, chain.block0)
    host = torch.empty(x.shape, dtype=x.dtype, pin_memory=True)
    host.copy_(x.cpu())
    n = x.numel()
    arena_bytes = 4 * n + 3 * n + (1 << 20)      # values + the stream (< 3 B/value here)
    arena = torch.empty(arena_bytes, dtype=torch.uint8, pin_memory=True)
    # (1) serial latency: one field at a time, every copy on the critical path
    ts = []
    bo = 0
    for _ in range(min(steps, 5) + 1):
        _flush(flush)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        xd = host.to(x.device, non_blocking=True)
        z, out, mean, var = chain.run(xd)
        sb, pb = z.totals()
        secs = [z.widths, z.outliers.view(torch.uint8), z.signs[:sb], z.payload[:pb], out.values]
        got = download_into(secs, arena, z.ctx)
        ts.append(time.perf_counter() - t0)
        bo = sum(g.size for g in got) + 16
        del z, out, xd, got
    t_serial = statistics.median(ts[1:])

    # (2) throughput: a three-stage pipeline over fields -- H2D of field k+1
    # (copy stream) | chain of field k (compute stream) | D2H of field k-1's
    # results (copy stream) -- so both PCIe directions and the SMs work at
    # once.  Every step still copies its whole input in and its whole result
    # out inside the timed region; nothing is reused between steps.
    dev = x.device
    s_in, s_cmp, s_out = (torch.cuda.Stream(device=dev) for _ in range(3))
    xin = [torch.empty_like(x), torch.empty_like(x)]
    arenas = [arena, torch.empty(arena_bytes, dtype=torch.uint8, pin_memory=True)]
    loaded = [None, None]      # H2D of slot j done
    consumed = [None, None]    # the chain finished reading xin[j]
    landed = [None, None]      # D2H into arenas[j] done
    keep = [None, None]        # device results of slot j, alive until their D2H lands

    def prefetch(j):
        with torch.cuda.stream(s_in):
            if consumed[j] is not None:
                s_in.wait_event(consumed[j])
            xin[j].copy_(host, non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(s_in)
            loaded[j] = ev

    def step(i, last):
        j = i % 2
        if not last:
            prefetch(1 - j)                           # next field's input streams in now
        with torch.cuda.stream(s_cmp):
            s_cmp.wait_event(loaded[j])
            z, out, mean, var = chain.run(xin[j])
            ev = torch.cuda.Event()
            ev.record(s_cmp)
            consumed[j] = ev
            sb, pb = z.totals()
        if landed[j] is not None:
            landed[j].synchronize()                   # arena j free; its old results released
        secs = (z.widths, z.outliers.view(torch.uint8), z.signs[:sb], z.payload[:pb],
                out.values.view(torch.uint8))
        with torch.cuda.stream(s_out):
            s_out.wait_event(consumed[j])
            off = 0
            for sec in secs:
                nb = sec.numel()
                arenas[j][off:off + nb].copy_(sec, non_blocking=True)
                sec.record_stream(s_out)
                off += (nb + 15) & ~15
            ev = torch.cuda.Event()
            ev.record(s_out)
            landed[j] = ev
        keep[j] = (z, out)
        return mean, var

    prefetch(0)
    for i in range(2):                                 # warm the streams' contexts
        step(i, last=(i == 1))
    torch.cuda.synchronize()
    if coll is not None:
        coll.barrier()
    # three timed passes of `steps` fields each; the median pass is reported
    # (one-off host or copy-engine hiccups move a single pass by tens of %)
    passes = []
    for _ in range(3):
        t0 = time.perf_counter()
        prefetch(0)                                    # every H2D is inside the timed region
        for i in range(steps):
            step(i, last=(i == steps - 1))
        for ev in landed:
            ev.synchronize()
        torch.cuda.synchronize()
        passes.append((time.perf_counter() - t0) / steps)
    keep[0] = keep[1] = None
    t = statistics.median(passes)
    if coll is not None:
        t = coll.max_over_ranks(t)
        t_serial = coll.max_over_ranks(t_serial)
    return {"value": round(len(OPS) * 4.0 * n_global / t / 1e9, 3), "unit": "GB/s",
            "ms_per_step": round(t * 1e3, 3), "h2d_bytes_per_step": 4 * n,
            "d2h_bytes_per_step": int(bo),
            "passes_ms_per_step": [round(v * 1e3, 3) for v in passes],
            "serial_ms_per_step": round(t_serial * 1e3, 3),
            "serial_value": round(len(OPS) * 4.0 * n_global / t_serial / 1e9, 3),
            "path": "pinned host field -> H2D -> public API chain -> D2H of the final stream "
                    "sections + decompressed field into pinned host arenas; pipelined over fields "
                    "on 3 CUDA streams (H2D of field k+1 | chain of field k | D2H of field k-1; "
                    "serial_*: one field at a time); h2d/d2h bytes are per rank"}


# ---------------------------------------------------------------------------
# CPU oracle arm (cpu_baseline and --impl reference)

_POOL_X = None


def _cpu_chain_slice(args):
    """Oracle op chain on one block-aligned slice [e0, e1) (fork-shared array)."""
    import hoszp_oracle as O

    e0, e1, eps, sadd, smul = args
    xs = _POOL_X[e0:e1]
    s = O.compress(xs, eps, (xs.size,), 32, "f32")
    z = O.scalar_mul(O.scalar_add(O.negate(s), sadd), smul)
    S, Q = O.moments(z)
    S2, _ = O.moments(z)           # mean and variance are separate passes in the reference
    O.decompress(z)
    return len(s["payload"]), S, Q


def _cpu_run(x, cfg, procs, eps=None):
    """One chain over `x` with `procs` worker processes (block-range slices).
    `eps` None: resolved from `x` (relative bound)."""
    import multiprocessing as mp

    global _POOL_X
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import hoszp_oracle as O

    _POOL_X = x
    t0 = time.perf_counter()
    if eps is None:
        eps = O.resolve_eps(x, cfg["rel_eps"], "rel")
    nb = -(-x.size // 32)
    from paper_2408_11971_b200.sharding import block_range

    jobs = []
    for r in range(procs):
        b0, b1 = block_range(nb, r, procs)
        jobs.append((b0 * 32, min(b1 * 32, x.size), eps, cfg["sadd"], cfg["smul"]))
    if procs == 1:
        res = [_cpu_chain_slice(j) for j in jobs]
    else:
        with mp.get_context("fork").Pool(procs) as pool:
            res = pool.map(_cpu_chain_slice, jobs)
    dt = time.perf_counter() - t0
    return dt, res


def _cpu_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def _cpu_baseline(x, cfg, budget_s=20.0):
    """Oracle chain on a bounded prefix sample of the same field, all cores."""
    procs = _cpu_cores()
    sample = min(x.size, max(32 * procs, 1 << 21))
    # grow the sample while the run stays inside the budget
    while True:
        dt, _ = _cpu_run(x[:sample], cfg, procs)
        if dt * 2.5 > budget_s or sample >= x.size:
            break
        sample = min(x.size, sample * 2)
    return {"value": round(len(OPS) * 4.0 * sample / dt / 1e9, 4), "unit": "GB/s",
            "cores": procs, "kind": "port", "os_cpu_count": os.cpu_count(),
            "affinity": len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else None,
            "sample": f"first {sample} of {x.size} values of the bench field (the same host "
                      f"array the B200 arm uploads), whole op chain, {procs} processes over "
                      f"block ranges ({dt:.2f} s)"}


def _reference_field(config):
    """The reference arm's input: the same values the B200 arm uses."""
    if config != 5:
        return host_field(config), "the whole field (the host array the B200 arm uploads)"
    import torch

    from paper_2408_11971_b200 import workloads as W

    # config 5 is generated on the GPU, slab by slab; the sample is a prefix of slab 0
    x = W.config5_slab(0, device="cuda:0")[: 1 << 27].cpu().numpy()
    torch.cuda.empty_cache()
    return x, "a prefix of slab 0 of the 2048^3 field (generated on cuda:0 exactly as the B200 arm)"


def run_reference(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    config = args.config or _default_config(world)
    cfg = W_cfg(config)
    x, origin = _reference_field(config)
    procs = _cpu_cores()
    # size the per-step sample so the whole --steps/--warmup run stays within
    # the budget: calibrate on a 2^22-value prefix, then scale
    cal = min(x.size, 1 << 22)
    dt, _ = _cpu_run(x[:cal], cfg, procs)
    per_elem = dt / cal
    budget_step = args.ref_budget / max(1, args.steps + args.warmup)
    sample = int(min(x.size, budget_step / per_elem))
    sample = max(32 * procs, (sample // (32 * procs)) * (32 * procs)) if sample < x.size else x.size
    xs = x[:sample]
    import hoszp_oracle as O

    eps = O.resolve_eps(x, cfg["rel_eps"], "rel")       # the field's eps, as in the B200 arm
    for _ in range(args.warmup):
        _cpu_run(xs, cfg, procs, eps=None if sample == x.size else eps)
    times = []
    for _ in range(args.steps):
        dt, _ = _cpu_run(xs, cfg, procs, eps=None if sample == x.size else eps)
        times.append(dt)
    t = sum(times) / len(times)
    value = len(OPS) * 4.0 * sample / t / 1e9
    gdims = _global_dims(config)
    what = (f"{sample} of {x.size} values: {origin}" if sample < x.size else origin)
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": "GB/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(t * 1e3, 3), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64 quantize / int64 bins (f32 input)",
        "data": "synthetic (seeded stand-in for SDRBench; see DESIGN.md)",
        "config": {"workload": f"config {config}: {'x'.join(map(str, gdims))} f32, rel eps "
                               f"{cfg['rel_eps']}, block_len 32, op chain {'>'.join(OPS)}, "
                               f"scalars sadd {cfg['sadd']} smul {cfg['smul']}",
                   "sample_elements": sample, "global_elements": _count(gdims)},
        "cpu_baseline": {"value": round(value, 4), "unit": "GB/s", "cores": procs, "kind": "port",
                         "os_cpu_count": os.cpu_count(),
                         "affinity": len(os.sched_getaffinity(0))
                         if hasattr(os, "sched_getaffinity") else None,
                         "sample": f"per step {what}; numpy oracle (oracle/hoszp_oracle.py, the "
                                   f"reference's algorithm restated) over {procs} processes"},
        "e2e": {"value": round(value, 4), "unit": "GB/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", type=int, default=None, choices=[2, 4, 5],
                    help="default: 4 at N = 1, 5 at N > 1")
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-scale-baseline", action="store_true",
                    help="skip the config-5 chain on one GPU (config5_n1) at N = 1")
    ap.add_argument("--quick", action="store_true",
                    help="functional run: chain timing + digests only (no kernel timing, e2e, "
                         "CPU baseline or config-5 scaling baseline)")
    ap.add_argument("--digest", action="store_true",
                    help="add digests of the whole-field streams / values (sharding check)")
    ap.add_argument("--cpu-budget", type=float, default=20.0)
    ap.add_argument("--ref-budget", type=float, default=200.0,
                    help="seconds of CPU work for the whole --impl reference run")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
