"""ctypes wrapper of oracle/bx_oracle.c -- TEST INFRASTRUCTURE ONLY.

Loads oracle/_build/libbx_oracle.so (built by ``make -C oracle`` or
``__graft_entry__.build()``).  The modulus table comes from the reference's own
table recorded in tests/golden/moduli.json, so the oracle never depends on the
product package.
"""
from __future__ import annotations

import ctypes
import json
import os
import pathlib
import subprocess

import numpy as np

HERE = pathlib.Path(__file__).resolve().parent
REPO = HERE.parent
LIB_PATH = HERE / "_build" / "libbx_oracle.so"

_lib = None
_mod = None


def build() -> pathlib.Path:
    subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            build()
        L = ctypes.CDLL(str(LIB_PATH))
        i64, i32, vp = ctypes.c_int64, ctypes.c_int, ctypes.c_void_p
        L.bxo_extract_eq.argtypes = [vp, i64, vp, i64, i32, i32, i64, vp, i32, vp, i64, i32, i32]
        L.bxo_extract_eq.restype = i32
        L.bxo_gf_mul.argtypes = [i32, vp, i32, vp, vp, vp, i64]
        L.bxo_gf_mul.restype = i32
        L.bxo_pack.argtypes = [vp, i32, i32, i64, vp]
        L.bxo_pack.restype = i32
        L.bxo_threads.restype = i32
        L.bxo_have_pclmul.restype = i32
        _lib = L
    return _lib


def moduli() -> dict[int, list[int]]:
    global _mod
    if _mod is None:
        raw = json.loads((REPO / "tests" / "golden" / "moduli.json").read_text())
        _mod = {int(k): v for k, v in raw.items()}
    return _mod


def _exps(q: int):
    e = moduli()[q]
    arr = (ctypes.c_int * len(e))(*e)
    return arr, len(e)


def _buf(data) -> tuple[np.ndarray, int]:
    a = np.frombuffer(data, dtype=np.uint8) if not isinstance(data, np.ndarray) else data
    a = np.ascontiguousarray(a.view(np.uint8))
    return a, a.ctypes.data


def threads() -> int:
    return int(lib().bxo_threads())


def extract_eq(x, y, q: int, n: int, nblocks: int, *, x_bit0: int = 0, y_bit0: int = 0,
               mode: int = 1, nthreads: int = 0) -> bytes:
    """Packed output bytes of `nblocks` equal-width blocks.

    mode 0 = literal reference algorithm (reduce every product), mode 1 = PCLMUL
    unreduced accumulation, mode 2 = mode 1 with byte-table / whole-element loads for
    byte-aligned q in {1,2,4,8,16,32,64} (bulk whole-stream checks);
    unreduced accumulation; both are pinned to the reference fixtures.
    """
    xa, xp = _buf(x)
    ya, yp = _buf(y)
    need = (max(x_bit0, y_bit0) + nblocks * q * n + 7) // 8
    if nblocks and (xa.size * 8 < x_bit0 + nblocks * q * n or ya.size * 8 < y_bit0 + nblocks * q * n):
        raise ValueError(f"streams too short for {nblocks} blocks ({need} bytes)")
    out = np.zeros((nblocks * q + 7) // 8 + 1, dtype=np.uint8)
    e, ne = _exps(q)
    rc = lib().bxo_extract_eq(xp, x_bit0, yp, y_bit0, q, n, nblocks, e, ne,
                              out.ctypes.data, 0, nthreads, mode)
    if rc:
        raise ValueError(f"bxo_extract_eq failed ({rc})")
    return out[: (nblocks * q + 7) // 8].tobytes()


def gf_mul(q: int, a: list[int], b: list[int]) -> list[int]:
    cnt = len(a)
    A = b"".join(int(v).to_bytes(16, "little") for v in a)
    Bb = b"".join(int(v).to_bytes(16, "little") for v in b)
    out = ctypes.create_string_buffer(16 * cnt)
    e, ne = _exps(q)
    rc = lib().bxo_gf_mul(q, e, ne, A, Bb, out, cnt)
    if rc:
        raise ValueError("bxo_gf_mul failed")
    raw = out.raw
    return [int.from_bytes(raw[16 * i:16 * i + 16], "little") for i in range(cnt)]


def pack(values, b: int) -> bytes:
    vals = [int(v) for v in values]
    words = 1 if b <= 64 else 2
    arr = np.zeros(len(vals) * words, dtype=np.uint64)
    for i, v in enumerate(vals):
        arr[i * words] = v & (2**64 - 1)
        if words == 2:
            arr[i * words + 1] = v >> 64
    nbytes = (len(vals) * b + 7) // 8
    out = np.zeros(nbytes + 1, dtype=np.uint8)
    rc = lib().bxo_pack(arr.ctypes.data, words, b, len(vals), out.ctypes.data)
    if rc:
        raise ValueError("bxo_pack failed")
    return out[:nbytes].tobytes()


def cpu_model() -> str:
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_count() -> int:
    return os.cpu_count() or 1
