"""Push-based streaming extraction over the native pipeline (bx_pipe_*).

For live producers: push the next bytes of both streams as they arrive and get
the packed output bytes of completed blocks back; partial blocks and the last
partial output byte carry over between pushes.

    with Pipe(q=4, n=64, chunk_bytes=64 << 20) as p:
        for xb, yb in capture():
            sink.write(p.push(xb, yb))
        sink.write(p.flush())

``depth`` pushes are kept in flight (default 2): a push enqueues its host
copy, H2D, kernel and D2H on the device and returns the output of the pushes
older than the newest ``depth - 1``, so push k+1's copies overlap push k's
kernel and D2H.  ``depth=1`` returns every push's own output (synchronous).
``flush`` returns everything still in flight plus the zero-padded last byte.
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from .errors import DeviceError


class Pipe:
    def __init__(self, q: int, n: int, chunk_bytes: int = 64 << 20, device: int = 0,
                 depth: int = 2):
        if not 1 <= q <= 128 or n < 1 or chunk_bytes < 1 or not 1 <= depth <= 4:
            raise ValueError("need 1 <= q <= 128, n >= 1, chunk_bytes >= 1, 1 <= depth <= 4")
        self.q, self.n, self.chunk, self.depth = q, n, chunk_bytes, depth
        L = _lib.lib()
        self._h = L.bx_pipe_create_async(q, n, chunk_bytes, device, depth)
        if not self._h:
            raise DeviceError("bx_pipe_create failed: "
                              + L.bx_last_error().decode(errors="replace"))
        # room for every retired push's output in one call (push or drain)
        self._cap = int(L.bx_pipe_max_output(self._h)) * depth
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
        """The output of every push still in flight, then the final partial
        output byte (zero padded), if any."""
        got = ctypes.c_int64()
        _lib.check(_lib.lib().bx_pipe_drain(self._h, self._out.ctypes.data, self._cap,
                                            ctypes.byref(got)), "bx_pipe_drain")
        rest = self._out[:got.value].tobytes()
        one = np.zeros(1, dtype=np.uint8)
        _lib.check(_lib.lib().bx_pipe_flush(self._h, one.ctypes.data, ctypes.byref(got)),
                   "bx_pipe_flush")
        return rest + one[:got.value].tobytes()

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
