"""ctypes binding of the C ABI declared in ``include/hsz_b200.h``.

The library is built in-tree (``_lib/libhsz_b200.so``, see ``build.py``).
There is no fallback: if the library is missing or the process has no CUDA
device, every operation raises.  Importing this module does not need a GPU
(the CPU test suite checks the exported symbols).
"""

from __future__ import annotations

import ctypes as C
import os

from . import build as _build

HSZ_OK = 0
HSZ_EINVAL = -1
HSZ_ECUDA = -2
HSZ_ETIMEDOUT = -3
HSZ_F32, HSZ_F64 = 0, 1
HSZ_OUT_F32, HSZ_OUT_F64, HSZ_OUT_BINS = 0, 1, 2
HSZ_OUT_BINS_ADD, HSZ_OUT_BINS_SUB = 3, 4
HSZ_TILE_BLOCKS = 128
HSZ_SECTION_SLACK = 16

_u8p = C.c_void_p
_vp = C.c_void_p
_u64 = C.c_uint64
_u32 = C.c_uint32
_i64 = C.c_int64
_int = C.c_int
_dbl = C.c_double

#: symbol -> (restype, argtypes); mirrors include/hsz_b200.h one-to-one
SIGNATURES = {
    "hsz_version": (C.c_char_p, []),
    "hsz_set_lookback_watchdog": (C.c_uint, [C.c_uint]),
    "hsz_set_host_wait_timeout": (C.c_double, [C.c_double]),
    "hsz_trace_read": (_int, [_vp, _int, _int]),
    "hsz_trace_lookback": (_int, [_vp]),
    "hsz_tile_count": (_u64, [_u64, _u32]),
    "hsz_sign_bound": (_u64, [_u64, _u32]),
    "hsz_payload_bound": (_u64, [_u64, _u32]),
    "hsz_workspace_size": (_u64, [_u64, _u32]),
    "hsz_workspace_init": (_int, [_vp, _u64, _vp]),
    "hsz_scalar_mul_scratch_size": (_u64, [_u64, _u32]),
    "hsz_minmax": (_int, [_vp, _int, _u64, _vp, _vp, _vp, _u64, _vp]),
    "hsz_compress": (_int, [_vp, _int, _u64, _u32, _dbl, _vp, _vp, _vp, _u64, _vp, _u64, _vp,
                            _vp, _vp, _u64, _vp]),
    "hsz_encode_bins": (_int, [_vp, _u64, _u32, _vp, _vp, _vp, _u64, _vp, _u64, _vp, _vp, _vp,
                               _u64, _vp]),
    "hsz_quantize": (_int, [_vp, _int, _u64, _dbl, _vp, _vp, _vp]),
    "hsz_dequantize": (_int, [_vp, _u64, _dbl, _int, _vp, _vp, _vp]),
    "hsz_tile_offsets": (_int, [_vp, _u64, _u32, _vp, _vp, _vp, _u64, _vp]),
    "hsz_decode": (_int, [_vp, _vp, _vp, _vp, _vp, _u64, _u32, _dbl, _int, _vp, _vp, _vp]),
    "hsz_negate": (_int, [_vp, _vp, _vp, _vp, _vp, _vp, _u64, _u32, _vp, _vp]),
    "hsz_scalar_add": (_int, [_vp, _vp, _u64, _i64, _vp, _vp]),
    "hsz_scalar_mul": (_int, [_vp, _vp, _vp, _vp, _vp, _u64, _u32, _dbl, _i64, _vp, _vp, _vp,
                              _u64, _vp, _u64, _vp, _vp, _vp, _vp, _u64, _vp]),
    "hsz_elementwise_scratch_size": (_u64, [_u64, _u32]),
    "hsz_elementwise": (_int, [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _u64, _u32, _int,
                               _vp, _vp, _vp, _u64, _vp, _u64, _vp, _vp, _vp, _vp, _u64, _vp]),
    "hsz_bivariate_scratch_size": (_u64, [_u64, _u32]),
    "hsz_hadamard": (_int, [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _u64, _u32, _dbl,
                            _vp, _vp, _vp, _u64, _vp, _u64, _vp, _vp, _vp, _vp, _u64, _vp]),
    "hsz_pair_stats": (_int, [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _u64, _u32, _vp,
                              _vp, _vp, _vp]),
    "hsz_block_means": (_int, [_vp, _vp, _vp, _vp, _vp, _u64, _u32, _dbl, _vp, _vp, _vp, _vp]),
    "hsz_moments": (_int, [_vp, _vp, _vp, _vp, _vp, _u64, _u32, _int, _vp, _vp, _vp, _u64, _vp]),
    "hsz_copy_d2h": (_int, [_vp, _vp, _u64, _vp]),
    "hsz_stream_sync": (_int, [_vp]),
    "hsz_fetch": (_int, [_vp, _vp, _u64, _vp]),
    "hsz_minmax_mb": (_int, [_vp, _int, _u64, _vp, _vp, _vp, _u64, _vp, _u64, _vp]),
    "hsz_moments_mb": (_int, [_vp, _vp, _vp, _vp, _vp, _u64, _u32, _int, _vp, _vp, _vp, _u64, _vp,
                              _u64, _vp]),
    "hsz_mailbox_wait": (_int, [_vp, _u64, _vp]),
    "hsz_hostcoll_bytes": (_u64, [_int]),
    "hsz_hostcoll_allgather": (_int, [_vp, _int, _int, _u64, _vp, _int, _vp, C.c_double]),
}

_LIB = None


class NativeLibraryMissing(RuntimeError):
    pass


def lib_path() -> str:
    return os.environ.get("HSZ_B200_LIB", _build.LIB)


def load(build_if_missing: bool = True):
    """Load (building first if needed) and return the ctypes library."""
    global _LIB
    if _LIB is not None:
        return _LIB
    path = lib_path()
    # HSZ_NO_BUILD=1: load exactly the given library (A/B runs of prebuilt variants)
    if os.environ.get("HSZ_NO_BUILD") == "1":
        build_if_missing = False
    if not os.path.exists(path) or (build_if_missing and _build.needs_build()):
        if not build_if_missing:
            raise NativeLibraryMissing(f"{path} not built; run python -m paper_2408_11971_b200.build")
        _build.build()
    lib = C.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _LIB = lib
    return lib


def check(rc: int, what: str) -> None:
    if rc == HSZ_ETIMEDOUT:
        from .errors import DeviceTimeout

        raise DeviceTimeout(f"{what}: the CUDA stream did not drain within the host wait bound "
                            "(a kernel hung; hsz_set_host_wait_timeout)")
    if rc != HSZ_OK:
        raise RuntimeError(f"{what} failed with status {rc} (invalid argument or CUDA launch error)")
