"""GF(2^256) block extraction -- config 3 as BASELINE states it (opt-in extension).

BASELINE config 3 asks for 1024-bit blocks with m = 256 output bits, i.e. a
field of q = 256 bits with n = 4 elements per block.  The reference caps the
field at q = 128 (`GFContext` raises `CapacityError`, pkg/src/blockext/
gf2q.py:20,111-112), so the drop-in API keeps that behaviour and this module
is the separate, explicitly-named path for q = 256 (SURVEY.md 8(d) C3
"optional extension").

The function is the reference's Ext_IP (extractor.py:77-87) applied to
consecutive disjoint q*n-bit windows (extractor.py:182-208, LSB-first elements,
bitio.py:45-60), with the modulus the reference's scan order picks for q = 256
(_moduli.py:1-11, restated in tools/gen_moduli.py): x^256 + x^10 + x^5 + x^2 + 1.
The output is the packed q-bit block results, LSB-first (bitio.py:74-88).
Computed by `bx_extract_eq_wide` (csrc/bx_wide.cu); no CPU fallback.
"""
from __future__ import annotations

import numpy as np

from .errors import CapacityError

WIDE_MODULI: dict[int, tuple[int, ...]] = {256: (256, 10, 5, 2, 0)}


def modulus_int(q: int) -> int:
    if q not in WIDE_MODULI:
        raise CapacityError(f"wide extraction supports q in {sorted(WIDE_MODULI)}, not {q}")
    v = 0
    for e in WIDE_MODULI[q]:
        v |= 1 << e
    return v


def extract_eq_wide(x, y, n: int, nblocks: int | None = None, *, q: int = 256,
                    device=None) -> bytes:
    """Packed outputs (q bits per block) of `nblocks` equal-width blocks read
    from bit 0 of x and y (bytes-like, numpy or torch tensors; CUDA tensors
    are used in place when 16-byte aligned).  nblocks defaults to as many
    whole blocks as both inputs hold."""
    import torch

    from . import _lib
    from . import device as D
    from .sharding import _as_tensor

    modulus_int(q)
    if n < 1:
        raise ValueError("vec_len must be >= 1")
    xt, yt = _as_tensor(x), _as_tensor(y)
    block_bytes = q * n // 8
    avail = min(xt.numel(), yt.numel()) // block_bytes
    if nblocks is None:
        nblocks = avail
    if nblocks < 0 or nblocks > avail:
        raise ValueError(f"{nblocks} blocks need {nblocks * block_bytes} bytes per stream; "
                         f"{min(xt.numel(), yt.numel())} available")
    if nblocks == 0:
        return b""
    dev = D.require_cuda(device if device is not None else (xt.device if xt.is_cuda else None))
    need = nblocks * block_bytes

    def on_device(t):
        if t.is_cuda and t.device == dev and t.data_ptr() % 16 == 0:
            return t
        buf, _ = D.to_device_stream(t[:need], dev)
        return buf

    xd, yd = on_device(xt), on_device(yt)
    out = torch.empty(nblocks * q // 32 + 4, dtype=torch.int32, device=dev)
    with torch.cuda.device(dev):
        _lib.check(_lib.lib().bx_extract_eq_wide(xd.data_ptr(), need, yd.data_ptr(), need, q, n,
                                                 nblocks, out.data_ptr(), 0,
                                                 D.stream_ptr(None, dev)), "bx_extract_eq_wide")
    return out.view(torch.uint8)[:nblocks * q // 8].cpu().numpy().tobytes()


def unpack_blocks(packed: bytes, q: int = 256) -> list[int]:
    """Block outputs as ints (LSB-first q-bit fields)."""
    a = np.frombuffer(packed, dtype=np.uint8)
    w = q // 8
    return [int.from_bytes(a[i * w:(i + 1) * w].tobytes(), "little") for i in range(len(a) // w)]


__all__ = ["WIDE_MODULI", "extract_eq_wide", "modulus_int", "unpack_blocks"]
