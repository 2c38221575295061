"""Pin config-scale parity to the REFERENCE itself: run the unmodified
reference package on the seeded BASELINE configs 1-4 (full size) and record
sha256 digests of everything the hot path produces.

Run in the build container (where ``/root/reference`` exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_ref_digests.py

It imports the reference from ``$HOSZP_REF_PATH`` (default
``/root/reference/pkg/src``) and writes ``tests/golden/ref_digests.json``.
Per config (and per eps of config 3's sweep) it records:

* ``field``     -- sha256 of the float32 input (workloads.py generators), so a
                   host whose generator output differs is reported as such;
* ``eps``       -- the reference's resolve_eps(rel) as float hex;
* ``compress``  -- sha256 of hoszp.serialize(hoszp.compress(...));
* ``negate`` / ``scalar_add`` / ``scalar_mul`` -- sha256 of the serialized
                   stream after each step of the chain
                   compress -> negate -> scalar_add -> scalar_mul;
* ``mean`` / ``variance`` -- ops.mean / ops.variance of the chain result
                   (float hex);
* ``decompress`` -- sha256 of the float32 bytes of decompress(chain result);
* ``decompress_compress`` -- sha256 of decompress(compress(...)).

The GPU test tests/test_gpu_ref_digests.py recomputes all of them through the
C ABI on a B200 and compares; nothing at test time reads /root/reference.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
REF = os.environ.get("HOSZP_REF_PATH", "/root/reference/pkg/src")
sys.path.insert(0, REF)
sys.path.insert(0, ROOT)
sys.dont_write_bytecode = True

import hoszp  # noqa: E402  (the reference)
from hoszp import ops  # noqa: E402

from paper_2408_11971_b200 import workloads as W  # noqa: E402  (generators only)

OUT = os.path.join(HERE, "ref_digests.json")


def sha(b) -> str:
    return hashlib.sha256(bytes(b)).hexdigest()


def cases():
    """(name, config, rel eps) of every pinned run."""
    out = [("config1", 1, W.CONFIGS[1]["rel_eps"]), ("config2", 2, W.CONFIGS[2]["rel_eps"])]
    for r in W.CONFIGS[3]["rel_sweep"]:
        out.append((f"config3_rel{r:g}", 3, r))
    out.append(("config4", 4, W.CONFIGS[4]["rel_eps"]))
    return out


def run_case(config: int, rel: float):
    cfg = W.CONFIGS[config]
    x = W.field(config)
    dims = tuple(cfg["dims"])
    raw = hoszp.RawArray(x, dims, "f32")
    eps = hoszp.resolve_eps(raw, rel, "rel")
    p = hoszp.QuantParams(eps, dims, 32, "f32")
    t0 = time.time()
    s = hoszp.compress(raw, p)
    d = {"field": sha(np.ascontiguousarray(x, dtype="<f4").tobytes()), "eps": float(eps).hex(),
         "dims": list(dims), "sadd": cfg["sadd"], "smul": cfg["smul"],
         "compress": sha(hoszp.serialize(s)),
         "decompress_compress": sha(np.asarray(hoszp.decompress(s).values, dtype="<f4").tobytes())}
    z = ops.negate(s)
    d["negate"] = sha(hoszp.serialize(z))
    z = ops.scalar_add(z, cfg["sadd"])
    d["scalar_add"] = sha(hoszp.serialize(z))
    z = ops.scalar_mul(z, cfg["smul"])
    d["scalar_mul"] = sha(hoszp.serialize(z))
    d["mean"] = float(ops.mean(z)).hex()
    d["variance"] = float(ops.variance(z)).hex()
    d["decompress"] = sha(np.asarray(hoszp.decompress(z).values, dtype="<f4").tobytes())
    d["reference_seconds"] = round(time.time() - t0, 1)
    return d


def main():
    out = {"generator": "tests/golden/make_ref_digests.py", "reference": REF,
           "numpy": np.__version__, "cases": {}}
    for name, config, rel in cases():
        t = time.time()
        out["cases"][name] = dict(config=config, rel_eps=rel, **run_case(config, rel))
        print(f"{name}: {time.time() - t:.1f} s", flush=True)
    with open(OUT, "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)
    print("wrote", OUT)


if __name__ == "__main__":
    main()
