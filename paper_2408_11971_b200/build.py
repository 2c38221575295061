"""Build the CUDA library in-tree (``_lib/libhsz_b200.so``) for sm_100a.

``python -m paper_2408_11971_b200.build`` or ``__graft_entry__.build()``.
The .so is git-ignored but travels to the GPU box with the repo snapshot.
"""

from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB_DIR = os.path.join(HERE, "_lib")
LIB = os.environ.get("HSZ_B200_LIB") or os.path.join(LIB_DIR, "libhsz_b200.so")
SOURCES = ["hsz_capi.cu"]
HEADERS = ["hsz_common.cuh", "hsz_quant.cuh", "hsz_k32.cuh", "hsz_generic.cuh", "hsz_enc32.cuh", "hsz_dec32.cuh",
           "hsz_bivar.cuh"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-shared", "-Xcompiler", "-fPIC",
    # no FMA contraction anywhere: the float64 quantizer must be bit-exact
    "-fmad=false",
]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.isabs(cand) and os.path.exists(cand) or not os.path.isabs(cand)):
            return cand
    return "nvcc"


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    deps.append(os.path.join(ROOT, "include", "hsz_b200.h"))
    return any(os.path.getmtime(p) > t for p in deps if os.path.exists(p))


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not needs_build():
        return LIB
    os.makedirs(LIB_DIR, exist_ok=True)
    extra = os.environ.get("HSZ_NVCC_EXTRA", "").split()   # experiments: -D knobs
    tmp = f"{LIB}.{os.getpid()}.tmp"     # concurrent builders (spawned ranks) do not collide
    cmd = [_nvcc(), *NVCC_FLAGS, *extra, "-o", tmp] + [os.path.join(CSRC, s) for s in SOURCES]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
        print(" ".join(cmd), flush=True)
    res = subprocess.run(cmd, capture_output=not verbose, text=True)
    if res.returncode != 0:
        sys.stderr.write((res.stdout or "") + (res.stderr or ""))
        raise RuntimeError(f"nvcc failed ({res.returncode}) building {LIB}")
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
