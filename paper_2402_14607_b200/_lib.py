"""ctypes binding of libbx_b200.so (the sm_100a kernels behind include/blockext_b200.h).

There is no CPU fallback: if the library is missing or cannot be loaded every
product entry point raises :class:`ExtensionMissingError`.
"""
from __future__ import annotations

import ctypes
import os
import pathlib
import threading

from .errors import CapacityError, DeviceError, ExtensionMissingError

_LIB_DIR = pathlib.Path(__file__).resolve().parent / "_lib"
#: BX_LIB=checked loads the bounds-checked build (see csrc/bx_core.cuh, BX_CHECK);
#: BX_LIB=/abs/path.so an experimental build (tools/build_variant.py)
_BX_LIB = os.environ.get("BX_LIB", "")
LIB_PATH = (pathlib.Path(_BX_LIB) if _BX_LIB.endswith(".so")
            else _LIB_DIR / ("libbx_b200_checked.so" if _BX_LIB == "checked" else "libbx_b200.so"))

BX_OK, BX_EINVAL, BX_ECUDA, BX_ERANGE = 0, -1, -2, -3

#: symbol -> (restype, argtypes); mirrors include/blockext_b200.h exactly
_i32, _i64, _vp, _cp = ctypes.c_int, ctypes.c_int64, ctypes.c_void_p, ctypes.c_char_p
_PI32, _PI64 = ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int64)
SIGNATURES = {
    "bx_version": (_i32, []),
    "bx_last_error": (_cp, []),
    "bx_modulus_exponents": (_i32, [_i32, _PI32]),
    "bx_extract_eq": (_i32, [_vp, _i64, _i64, _vp, _i64, _i64, _i32, _i32, _i64, _vp, _i64, _vp]),
    "bx_extract_neq": (_i32, [_vp, _i64, _vp, _i64, _i32, _i32, _i32, _i64, _vp, _vp]),
    "bx_launch_info": (_i32, [_i32, _i32, _i64, _PI32, _PI32, _PI32, _PI32, _PI32, _PI64, _PI32]),
    "bx_pack": (_i32, [_vp, _i32, _i32, _i64, _vp, _i64, _vp]),
    "bx_launch_count": (_i64, [_i32]),
    "bx_checked_violations": (_i64, [_i32, _PI64]),
    "bx_gf_ip_generic": (_i32, [_i32, _vp, _vp, _vp, _i32, _i64, _vp, _vp]),
    "bx_pipe_create": (_vp, [_i32, _i32, _i64, _i32]),
    "bx_pipe_push": (_i32, [_vp, _vp, _vp, _i64, _vp, _i64, _PI64]),
    "bx_pipe_flush": (_i32, [_vp, _vp, _PI64]),
    "bx_pipe_create_async": (_vp, [_i32, _i32, _i64, _i32, _i32]),
    "bx_gf_pow": (_i32, [_i32, _vp, _vp, _vp, _i64, _vp, _vp]),
    "bx_extract_eq_wide": (_i32, [_vp, _i64, _vp, _i64, _i32, _i32, _i64, _vp, _i64, _vp]),
    "bx_extract_eq_host": (_i32, [_vp, _i64, _i64, _vp, _i64, _i64, _i32, _i32, _i64, _vp, _i32]),
    "bx_pipe_drain": (_i32, [_vp, _vp, _i64, _PI64]),
    "bx_pipe_max_output": (_i64, [_vp]),
    "bx_pipe_blocks": (_i64, [_vp]),
    "bx_pipe_destroy": (None, [_vp]),
    "bx_bernoulli_bits": (_i32, [_vp, _i64, ctypes.c_double, ctypes.c_uint64, _i64, _vp]),
    "bx_xor_scan_scratch_bytes": (_i64, [_i64, _i32]),
    "bx_xor_scan_rows": (_i32, [_vp, _i64, _i32, _vp, _vp]),
    "bx_markov_scratch_bytes": (_i64, [_i64, _i32]),
    "bx_markov_chain": (_i32, [_vp, _i64, _vp, _i32, _i32, _vp, _vp, _vp]),
    "bx_ip_table": (_i32, [_i32, _i32, ctypes.c_uint32, ctypes.c_uint32, _vp, _vp]),
    "bx_ip_histograms": (_i32, [_i32, _i32, ctypes.c_uint32, ctypes.c_uint32, _vp, _vp]),
    "bx_rows_uniform": (_i32, [_vp, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32, _vp, _vp]),
}

_lock = threading.Lock()
_handle = None


def lib():
    """The loaded library (loaded once); raises ExtensionMissingError if absent."""
    global _handle
    if _handle is not None:
        return _handle
    with _lock:
        if _handle is None:
            if not LIB_PATH.exists():
                raise ExtensionMissingError(
                    f"{LIB_PATH} is not built; run `python -m paper_2402_14607_b200.build` "
                    "(there is no CPU fallback)")
            try:
                h = ctypes.CDLL(str(LIB_PATH))
            except OSError as exc:
                raise ExtensionMissingError(f"cannot load {LIB_PATH}: {exc}") from exc
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(h, name)
                fn.restype = res
                fn.argtypes = args
            _handle = h
    return _handle


def check(rc: int, what: str) -> int:
    if rc >= 0:
        return rc
    msg = lib().bx_last_error().decode(errors="replace")
    if rc == BX_ERANGE:
        raise CapacityError(f"{what}: {msg}")
    if rc == BX_EINVAL:
        raise ValueError(f"{what}: {msg}")
    raise DeviceError(f"{what}: {msg}")


def modulus_exponents(q: int) -> tuple[int, ...]:
    buf = (ctypes.c_int * 5)()
    cnt = check(lib().bx_modulus_exponents(q, buf), "bx_modulus_exponents")
    return tuple(buf[:cnt])


def launch_info(q: int, n: int, nblocks: int) -> dict:
    vals = [ctypes.c_int() for _ in range(6)]
    grid = ctypes.c_int64()
    fam = ctypes.c_int()
    check(lib().bx_launch_info(q, n, nblocks, *[ctypes.byref(v) for v in vals[:5]],
                               ctypes.byref(grid), ctypes.byref(fam)), "bx_launch_info")
    tpb, tile, staged, threads, smem = (v.value for v in vals[:5])
    return {"tpb": tpb, "tile": tile, "staged": staged, "threads": threads,
            "smem_bytes": smem, "grid": grid.value,
            "family": ("diag", "holes")[fam.value & 1], "direct": bool(fam.value & 2),
            "tma": bool(fam.value & 4)}


def launch_count(reset: bool = False) -> int:
    return int(lib().bx_launch_count(1 if reset else 0))


def checked_violations(reset: bool = False) -> tuple[int, tuple[int, int, int]]:
    """(count, (tag, index, bound) of the first) from a BX_CHECKED build; -1 otherwise."""
    first = (ctypes.c_int64 * 3)()
    n = int(lib().bx_checked_violations(1 if reset else 0, first))
    return n, tuple(first)
