"""Push-based streaming extraction over the native pipeline (bx_pipe_*).

For live producers: push the next bytes of both streams as they arrive and get
the packed output bytes of every block completed so far; partial blocks and
the last partial output byte carry over between pushes.

    with Pipe(q=4, n=64, chunk_bytes=64 << 20) as p:
        for xb, yb in capture():
            sink.write(p.push(xb, yb))
        sink.write(p.flush())
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from .errors import DeviceError


class Pipe:
    def __init__(self, q: int, n: int, chunk_bytes: int = 64 << 20, device: int = 0):
        if not 1 <= q <= 128 or n < 1 or chunk_bytes < 1:
            raise ValueError("need 1 <= q <= 128, n >= 1, chunk_bytes >= 1")
        self.q, self.n, self.chunk = q, n, chunk_bytes
        self._h = _lib.lib().bx_pipe_create(q, n, chunk_bytes, device)
        if not self._h:
            raise DeviceError("bx_pipe_create failed (no device or out of memory)")
        # enough for the outputs of one push: blocks in (chunk + carried) bytes
        self._cap = (8 * (chunk_bytes + (q * n + 7) // 8 + 1) // (q * n)) * q // 8 + 2
        self._out = np.empty(self._cap, dtype=np.uint8)

    def push(self, x, y) -> bytes:
        """Feed the next bytes of both streams (equal lengths, <= chunk_bytes)."""
        xa = np.frombuffer(memoryview(x), dtype=np.uint8)
        ya = np.frombuffer(memoryview(y), dtype=np.uint8)
        if xa.size != ya.size:
            raise ValueError("push equal byte counts of both streams")
        if xa.size > self.chunk:
            raise ValueError(f"push at most {self.chunk} bytes per stream")
        got = ctypes.c_int64()
        _lib.check(_lib.lib().bx_pipe_push(self._h, xa.ctypes.data, ya.ctypes.data, xa.size,
                                           self._out.ctypes.data, self._cap, ctypes.byref(got)),
                   "bx_pipe_push")
        return self._out[:got.value].tobytes()

    def flush(self) -> bytes:
        """The final partial output byte (zero padded), if any."""
        one = np.zeros(1, dtype=np.uint8)
        got = ctypes.c_int64()
        _lib.check(_lib.lib().bx_pipe_flush(self._h, one.ctypes.data, ctypes.byref(got)),
                   "bx_pipe_flush")
        return one[:got.value].tobytes()

    @property
    def blocks(self) -> int:
        return int(_lib.lib().bx_pipe_blocks(self._h))

    def close(self) -> None:
        if self._h:
            _lib.lib().bx_pipe_destroy(self._h)
            self._h = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()
        return False

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001 - interpreter shutdown
            pass
