"""Device-buffer layer over the C ABI: torch tensors as HBM buffers, CUDA streams.

PyTorch is plumbing here (allocation, streams, copies); all compute is the
sm_100a library.  Stream buffers are uint8 tensors padded so the kernels may
read whole 32-bit words plus one guard word past the last stream bit.
"""
from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .errors import DeviceError

PAD_BYTES = 16


def require_cuda(device=None) -> torch.device:
    if not torch.cuda.is_available():
        raise DeviceError("no CUDA device: the extractor runs only on the sm_100a kernels")
    if device is None:
        return torch.device("cuda", torch.cuda.current_device())
    d = torch.device(device)
    if d.type != "cuda":
        raise DeviceError(f"device {d} is not a CUDA device")
    return d if d.index is not None else torch.device("cuda", torch.cuda.current_device())


def padded_len(nbytes: int) -> int:
    return ((nbytes + 15) // 16) * 16 + PAD_BYTES


def empty_stream(nbytes: int, device, zero_pad: bool = True) -> torch.Tensor:
    """uint8 device buffer for `nbytes` of stream data plus the guard padding."""
    t = torch.empty(padded_len(nbytes), dtype=torch.uint8, device=device)
    if zero_pad:
        t[nbytes:].zero_()
    return t


def to_device_stream(data, device, pin: bool = False) -> tuple[torch.Tensor, int]:
    """Copy host bytes-like / numpy / torch data into a padded device buffer."""
    if isinstance(data, torch.Tensor):
        src = data.reshape(-1).view(torch.uint8)
    else:
        arr = np.frombuffer(memoryview(data), dtype=np.uint8) if not isinstance(data, np.ndarray) \
            else np.ascontiguousarray(data).reshape(-1).view(np.uint8)
        if arr.size:
            import warnings
            with warnings.catch_warnings():   # read-only source buffers are only read
                warnings.simplefilter("ignore")
                src = torch.from_numpy(arr)
        else:
            src = torch.empty(0, dtype=torch.uint8)
        if pin and src.numel():
            src = src.pin_memory()
    n = src.numel()
    buf = empty_stream(n, device)
    if n:
        buf[:n].copy_(src, non_blocking=pin)
    return buf, n


def stream_ptr(stream: torch.cuda.Stream | None = None, device=None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream(device)
    return int(s.cuda_stream)


def extract_eq(x: torch.Tensor, x_bytes: int, y: torch.Tensor, y_bytes: int, q: int, n: int,
               nblocks: int, *, x_bit0: int = 0, y_bit0: int = 0, out: torch.Tensor | None = None,
               out_bit0: int = 0, stream: torch.cuda.Stream | None = None) -> torch.Tensor:
    """Launch bx_extract_eq on device buffers; returns the (padded) output buffer."""
    if out is None:
        nbytes = (out_bit0 + nblocks * q + 7) // 8
        out = torch.zeros(padded_len(nbytes), dtype=torch.uint8, device=x.device)
    for t in (x, y, out):
        if not t.is_cuda or t.dtype != torch.uint8 or not t.is_contiguous():
            raise ValueError("device buffers must be contiguous uint8 CUDA tensors")
    # no torch.cuda.device() context: the library selects the device that owns
    # x itself (DeviceScope in bx_abi.cu), which keeps small launches cheap
    rc = _lib.lib().bx_extract_eq(x.data_ptr(), x_bytes, x_bit0, y.data_ptr(), y_bytes, y_bit0,
                                  q, n, nblocks, out.data_ptr(), out_bit0,
                                  stream_ptr(stream, x.device))
    if rc:
        _lib.check(rc, "bx_extract_eq")
    return out


def pack(samples: torch.Tensor, b: int, *, out: torch.Tensor | None = None, out_bit0: int = 0,
         stream: torch.cuda.Stream | None = None) -> torch.Tensor:
    """Pack the low b bits of each sample LSB-first (reference sources.py:116-121)."""
    elem = samples.element_size()
    if elem not in (1, 2, 4, 8) or samples.is_floating_point():
        raise ValueError("samples must be an integer tensor of 1, 2, 4 or 8 byte elements")
    if not 1 <= b <= 8 * elem:
        raise ValueError(f"bits per sample {b} outside 1..{8 * elem}")
    nat = 1 if b <= 8 else 2 if b <= 16 else 4 if b <= 32 else 8
    if elem > nat and not (elem == 2 and b <= 8) and samples.numel() >= 4096:
        # keep the low `nat` bytes of every (little-endian) sample so the tile
        # kernel for the natural type runs: an exact bit slice, not a cast
        narrow = {1: torch.uint8, 2: torch.int16, 4: torch.int32}[nat]
        samples = samples.contiguous().view(narrow).view(-1, elem // nat)[:, 0].contiguous()
        elem = nat
    count = samples.numel()
    if out is None:
        end = out_bit0 + count * b
        out = empty_stream((end + 7) // 8, samples.device)
        out[(end // 32) * 4:].zero_()   # zero pad bits of the last word (bitio.py:84-88)
    with torch.cuda.device(samples.device):
        _lib.check(_lib.lib().bx_pack(samples.data_ptr(), elem, b, count, out.data_ptr(), out_bit0,
                                      stream_ptr(stream, samples.device)), "bx_pack")
    return out


def extract_neq(x: torch.Tensor, x_bytes: int, y: torch.Tensor, y_bytes: int, q1: int, step: int,
                n: int, nblocks: int, *, out: torch.Tensor | None = None,
                stream: torch.cuda.Stream | None = None) -> torch.Tensor:
    """Launch bx_extract_neq (widths q1 + k*step) on device buffers."""
    total = sum(q1 + k * step for k in range(nblocks))
    if out is None:
        out = torch.zeros(padded_len((total + 7) // 8), dtype=torch.uint8, device=x.device)
    with torch.cuda.device(x.device):
        _lib.check(_lib.lib().bx_extract_neq(x.data_ptr(), x_bytes, y.data_ptr(), y_bytes, q1, step,
                                             n, nblocks, out.data_ptr(), stream_ptr(stream, x.device)),
                   "bx_extract_neq")
    return out


def bernoulli_bits(nbits: int, p: float, seed: int, *, bit0: int = 0, out: torch.Tensor | None = None,
                   out_byte0: int = 0, device=None, stream=None) -> torch.Tensor:
    """Counter-based Bernoulli(p) bits [bit0, bit0+nbits) (bx_bernoulli_bits), written at
    byte out_byte0 of `out` (4-byte aligned offset)."""
    dev = require_cuda(device) if out is None else out.device
    if out is None:
        out = empty_stream((nbits + 7) // 8, dev)
    if out_byte0 % 4:
        raise ValueError("out_byte0 must be a multiple of 4")
    with torch.cuda.device(dev):
        _lib.check(_lib.lib().bx_bernoulli_bits(out.data_ptr() + out_byte0, nbits, float(p),
                                                int(seed) & (2**64 - 1), bit0,
                                                stream_ptr(stream, dev)), "bx_bernoulli_bits")
    return out


def xor_scan_rows(buf: torch.Tensor, rows: int, row_bytes: int, stream=None) -> torch.Tensor:
    """In place: row r of the (rows x row_bytes) byte matrix := XOR of rows 0..r."""
    if row_bytes % 4 or buf.data_ptr() % 4:
        raise ValueError("rows must be whole, aligned 32-bit words")
    L = _lib.lib()
    words = row_bytes // 4
    scratch = torch.empty(max(4, _lib.check(L.bx_xor_scan_scratch_bytes(rows, words), "scratch")),
                          dtype=torch.uint8, device=buf.device)
    with torch.cuda.device(buf.device):
        _lib.check(L.bx_xor_scan_rows(buf.data_ptr(), rows, words, scratch.data_ptr(),
                                      stream_ptr(stream, buf.device)), "bx_xor_scan_rows")
    return buf


def markov_chain(u: torch.Tensor, cum: torch.Tensor, b: int, start: int, stream=None) -> torch.Tensor:
    """Reference markov sample path on the device (bx_markov_chain); int16 states."""
    if u.dtype != torch.float64 or cum.dtype != torch.float64 or not u.is_cuda or not cum.is_cuda:
        raise ValueError("u and cum must be float64 CUDA tensors")
    L = _lib.lib()
    count = u.numel()
    vals = torch.empty(count, dtype=torch.int16, device=u.device)
    scratch = torch.empty(max(4, _lib.check(L.bx_markov_scratch_bytes(count, b), "scratch")),
                          dtype=torch.uint8, device=u.device)
    with torch.cuda.device(u.device):
        _lib.check(L.bx_markov_chain(u.data_ptr(), count, cum.data_ptr(), b, start, vals.data_ptr(),
                                     scratch.data_ptr(), stream_ptr(stream, u.device)),
                   "bx_markov_chain")
    return vals
