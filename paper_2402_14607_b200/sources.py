"""Seeded source simulators with the reference's semantics, packed on the GPU.

Mirrors reference pkg/src/blockext/sources.py:36-167 for the parts on the hot
path: model constructors, ``generate`` and the
sample packer ``_pack_samples``.  The random draws stay numpy PCG64
(``default_rng(seed)``, one 64-bit step per sample) so streams are
byte-identical to the reference; mapping draws to samples (threshold or
inverse-CDF search) and packing samples into the LSB-first bit stream run on
the device (``bx_pack``, reference sources.py:116-121).

Min-entropy certification (sources.py:170-234) is host analytics outside the
data path and is not re-implemented here (out of scope).
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Sequence

import numpy as np

from .errors import TruncatedSourceError

PROB_SUM_TOL = 2.0 ** -30
DRAW_CHUNK = 1 << 24


@dataclass(frozen=True)
class SourceModel:
    """A (b, N, rate)-block source specification (reference sources.py:36-50)."""

    kind: str
    bits_per_sample: int
    seed: int = 0
    p: float | None = None
    table: np.ndarray | None = None
    path: str | None = None


def _check_distribution(probs, what: str) -> np.ndarray:
    probs = np.asarray(probs, dtype=np.float64)
    if np.any(probs < 0):
        raise ValueError(f"{what} has negative entries")
    if abs(float(probs.sum()) - 1.0) > PROB_SUM_TOL:
        raise ValueError(f"{what} sums to {probs.sum()!r}, not 1 within 2^-30")
    return probs


def iid_biased(p: float, seed: int = 0) -> SourceModel:
    if not 0.0 <= p <= 1.0:
        raise ValueError(f"bias {p} outside [0,1]")
    return SourceModel(kind="iid-biased", bits_per_sample=1, seed=seed, p=p)


def iid_table(probs: Sequence[float], bits_per_sample: int, seed: int = 0) -> SourceModel:
    probs = _check_distribution(np.asarray(probs), "probability table")
    if probs.shape != (1 << bits_per_sample,):
        raise ValueError(f"table length {probs.shape} does not match 2^{bits_per_sample} outcomes")
    return SourceModel(kind="iid-table", bits_per_sample=bits_per_sample, seed=seed, table=probs)


def markov(transitions, bits_per_sample: int, seed: int = 0) -> SourceModel:
    t = np.asarray(transitions, dtype=np.float64)
    size = 1 << bits_per_sample
    if t.shape != (size, size):
        raise ValueError(f"transition table must be {size}x{size}, got {t.shape}")
    for row in range(size):
        _check_distribution(t[row], f"transition row {row}")
    return SourceModel(kind="markov", bits_per_sample=bits_per_sample, seed=seed, table=t)


def file_source(path: str, bits_per_sample: int) -> SourceModel:
    return SourceModel(kind="file", bits_per_sample=bits_per_sample, path=path)


# ------------------------------------------------------------ device side

def _sample_dtype(b: int):
    import torch
    return torch.uint8 if b <= 8 else torch.int16 if b <= 16 else torch.int32 if b <= 32 else torch.int64


def generate_device(model: SourceModel, count: int, device=None):
    """Packed stream of `count` samples as a padded uint8 device buffer.

    Returns (buffer, nbytes).  Identical bytes to reference ``generate``.
    """
    import torch

    from . import device as D

    if count < 1:
        raise ValueError("sample count must be >= 1")
    dev = D.require_cuda(device)
    b = model.bits_per_sample
    nbytes = (count * b + 7) // 8
    if model.kind == "file":
        need_bits = count * b
        with open(model.path, "rb") as fh:
            data = fh.read(nbytes)
        if len(data) < nbytes:
            raise TruncatedSourceError(
                f"{model.path} holds {len(data)} bytes; {nbytes} needed for {count} samples of {b} bits")
        buf = bytearray(data)
        if need_bits % 8:
            buf[-1] &= (1 << (need_bits % 8)) - 1
        return D.to_device_stream(bytes(buf), dev)
    rng = np.random.default_rng(model.seed)
    out = D.empty_stream(nbytes, dev)
    out[(count * b // 32) * 4:].zero_()
    if model.kind == "iid-biased":
        # reference sources.py:133-136: bit = random() < p
        for s in range(0, count, DRAW_CHUNK):
            c = min(DRAW_CHUNK, count - s)
            u = torch.from_numpy(rng.random(c)).to(dev, non_blocking=False)
            bits = (u < model.p).to(torch.uint8)
            D.pack(bits, 1, out=out, out_bit0=s)
        return out, nbytes
    if model.kind == "iid-table":
        # reference sources.py:137-140: rng.choice(len(table), size, p=table), i.e.
        # numpy's inverse-CDF search: cdf = cumsum(p) / cdf[-1]; searchsorted(right)
        cdf = np.cumsum(model.table)
        cdf /= cdf[-1]
        cdf_d = torch.from_numpy(cdf).to(dev)
        dt = _sample_dtype(b)
        for s in range(0, count, DRAW_CHUNK):
            c = min(DRAW_CHUNK, count - s)
            u = torch.from_numpy(rng.random(c)).to(dev)
            vals = torch.searchsorted(cdf_d, u, right=True).to(dt)
            D.pack(vals, b, out=out, out_bit0=s * b)
        return out, nbytes
    if model.kind == "markov":
        # reference sources.py:141-152: u = random(count), then the start state
        # integers(0, 2^b); the chain itself runs on the device
        # (bx_markov_chain, segmented parallel walk), then bx_pack.
        if b > 16:
            raise ValueError("markov models are limited to b <= 16 on the device")
        cum = np.cumsum(model.table, axis=1)
        cum[:, -1] = 1.0
        u = torch.from_numpy(rng.random(count)).to(dev)
        state = int(rng.integers(0, 1 << b))
        vals = D.markov_chain(u, torch.from_numpy(cum).to(dev), b, state)
        D.pack(vals, b, out=out)
        return out, nbytes
    raise ValueError(f"cannot generate from a {model.kind!r} model")


def generate(model: SourceModel, count: int) -> bytes:
    """Deterministic sample stream: count samples packed little-endian
    (reference sources.py:124-167); byte-identical output."""
    buf, nbytes = generate_device(model, count)
    return buf[:nbytes].cpu().numpy().tobytes()


def _pack_samples(values, bits_per_sample: int) -> bytes:
    """Low b bits of each value, LSB-first (reference sources.py:116-121), on the GPU."""
    import torch

    from . import device as D

    dev = D.require_cuda()
    b = bits_per_sample
    arr = np.asarray(values).astype(np.uint64, copy=False)
    if b < 64:
        # the low b bits in the narrowest type that holds them (less H2D, and
        # the packer's tile kernel for that type)
        nat = np.uint8 if b <= 8 else np.uint16 if b <= 16 else np.uint32 if b <= 32 else np.uint64
        arr = (arr & np.uint64((1 << b) - 1)).astype(nat)
    t = torch.from_numpy(np.ascontiguousarray(arr).view(np.dtype(f"i{arr.itemsize}")) if arr.itemsize > 1
                         else np.ascontiguousarray(arr)).to(dev)
    nbytes = (arr.size * b + 7) // 8
    return D.pack(t, b)[:nbytes].cpu().numpy().tobytes()


__all__ = ["SourceModel", "file_source", "generate", "generate_device", "iid_biased",
           "iid_table", "markov"]
