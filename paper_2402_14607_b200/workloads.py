"""Seeded synthetic workloads for the five BASELINE.json configs.

Every stream is produced exactly the way the reference's ``generate`` produces it
(reference pkg/src/blockext/sources.py:124-152): ``numpy.random.default_rng(seed)``
(PCG64), one 64-bit draw per sample, so

* ``iid-biased(p)``  -> ``rng.random(count) < p``, bits packed LSB-first (:133-136)
* ``iid-table(pmf)`` -> ``rng.choice(len(pmf), size=count, p=pmf)`` (:137-140)

Because each sample costs exactly one PCG64 step, the window of block ``l`` can
be regenerated on its own with ``bit_generator.advance`` -- that is how the golden
fixtures pin sampled blocks of the full-size configs against the reference.

The block-Markov source of config 4 has no reference generator (the reference
``markov`` kind is a per-sample chain, sources.py:141-152); it is defined here:
block 0 uniform, block k = block k-1 XOR a Bernoulli(0.2) mask.

Nothing here touches the GPU; the device-side generators live in ``sources``.
"""
from __future__ import annotations

import math
import os
from dataclasses import dataclass

import numpy as np

ADC_MEAN = 128.0
ADC_SIGMA = 20.0


def adc_pmf(mean: float = ADC_MEAN, sigma: float = ADC_SIGMA) -> np.ndarray:
    """pmf of an 8-bit ADC sampling N(mean, sigma^2), rounded and clipped to 0..255."""
    def cdf(v: float) -> float:
        return 0.5 * (1.0 + math.erf((v - mean) / (sigma * math.sqrt(2.0))))

    edges = [cdf(k + 0.5) for k in range(255)]
    p = np.empty(256, dtype=np.float64)
    p[0] = edges[0]
    for k in range(1, 255):
        p[k] = edges[k] - edges[k - 1]
    p[255] = 1.0 - edges[254]
    return p


UNIFORM8 = np.full(256, 1.0 / 256.0)


@dataclass(frozen=True)
class SourceSpec:
    """One synthetic stream: kind in {"iid-biased", "iid-table", "block-markov"}."""

    kind: str
    seed: int
    bits_per_sample: int
    p: float = 0.5                     # iid-biased: P(bit = 1); block-markov: flip prob.
    table: tuple | None = None         # iid-table pmf (hashable copy)
    block_bits: int = 0                # block-markov: bits per chained block

    def pmf(self) -> np.ndarray:
        return np.asarray(self.table, dtype=np.float64)


def iid_biased_spec(p: float, seed: int) -> SourceSpec:
    return SourceSpec("iid-biased", seed, 1, p=p)


def adc_spec(seed: int) -> SourceSpec:
    return SourceSpec("iid-table", seed, 8, table=tuple(adc_pmf().tolist()))


def uniform8_spec(seed: int) -> SourceSpec:
    return SourceSpec("iid-table", seed, 8, table=tuple(UNIFORM8.tolist()))


def block_markov_spec(flip: float, seed: int, block_bits: int) -> SourceSpec:
    return SourceSpec("block-markov", seed, 1, p=flip, block_bits=block_bits)


@dataclass(frozen=True)
class Workload:
    name: str
    q: int                 # field bits (output bits per block)
    n: int                 # vec_len (elements per block)
    samples: int           # samples per source
    x: SourceSpec
    y: SourceSpec
    note: str = ""
    entropy_rate: tuple = (3, 4)  # per sample bit, as a fraction (num, den)

    @property
    def b(self) -> int:
        return self.x.bits_per_sample

    @property
    def block_bits(self) -> int:
        return self.q * self.n

    @property
    def num_blocks(self) -> int:
        return self.samples * self.b // self.block_bits

    @property
    def stream_bytes(self) -> int:
        return (self.samples * self.b + 7) // 8

    def plan(self):
        """EqPlan for this workload (hand-assembled like the reference tests'
        ``tiny_eq_plan``, pkg/tests/test_extractor.py:32-38)."""
        from fractions import Fraction

        from .params import EqPlan, error_bound_eq

        rate = Fraction(*self.entropy_rate)
        draft = EqPlan(self.b, self.samples, rate, Fraction(1, 2), self.n, self.q,
                       self.num_blocks, self.num_blocks * self.q, 0.0)
        return EqPlan(**{**draft.__dict__, "log2_error": error_bound_eq(draft)})


def _c5(n_bits: int) -> Workload:
    q = n_bits // 64
    return Workload(f"c5_n{n_bits}", q, 64, 2**33, uniform8_spec(1), adc_spec(2),
                    note=f"2^36-bit uniform x / ADC y, block {n_bits} bits, q=n/64")


WORKLOADS: dict[str, Workload] = {
    "c1": Workload("c1", 32, 4, 2**20, iid_biased_spec(0.5, 1), iid_biased_spec(0.5, 2),
                   note="CPU-runnable oracle config: 2x2^20 uniform bits, 128-bit blocks",
                   entropy_rate=(1, 1)),
    "c2": Workload("c2", 4, 64, 2**28, adc_spec(1), adc_spec(2),
                   note="vacuum-noise QRNG: 2x2^28 8-bit ADC samples N(128,20), 256-bit blocks"),
    "c2p": Workload("c2p", 56, 48, 2**28, adc_spec(1), adc_spec(2),
                    note="config 2 through the planner: plan_eq(8, 2^28, 3/4, 2^-30)"),
    "c3": Workload("c3", 128, 8, 2**32, iid_biased_spec(0.3, 1), iid_biased_spec(0.3, 2),
                   note="large blocks: 2x2^32 Bernoulli(0.3) bits, 1024-bit blocks, m=128"),
    "c4": Workload("c4", 4, 128, 2**34,
                   block_markov_spec(0.2, 1, 512), block_markov_spec(0.2, 2, 512),
                   note="forward-block stress: 512-bit blocks, block-Markov flip 0.2"),
    "c4p": Workload("c4p", 58, 120, 2**34,
                    block_markov_spec(0.2, 1, 512), block_markov_spec(0.2, 2, 512),
                    note="config 4 planner shape (6960-bit blocks, not word aligned)"),
    "c5_n128": _c5(128),
    "c5_n256": _c5(256),
    "c5_n512": _c5(512),
    "c5_n1024": _c5(1024),
    "c5_n2048": _c5(2048),
    "paper": Workload("paper", 80, 71, 2**28, uniform8_spec(1), uniform8_spec(2),
                      note="paper flagship shape q=80, n=71 (PAPER.md:268-270); 2x256 MiB "
                           "streams like config 2 (a steady-state stream, larger than L2)"),
}


# ------------------------------------------------------------------ host RNG --

def _samples_iid(spec: SourceSpec, start: int, count: int) -> np.ndarray:
    """Samples [start, start+count) of an iid stream, one PCG64 step per sample."""
    rng = np.random.default_rng(spec.seed)
    if start:
        rng.bit_generator.advance(start)
    if spec.kind == "iid-biased":
        return (rng.random(count) < spec.p).astype(np.uint8)
    if spec.kind == "iid-table":
        return rng.choice(len(spec.table), size=count, p=spec.pmf()).astype(np.uint8)
    raise ValueError(f"not an iid kind: {spec.kind}")


def _pack_bits_host(bits: np.ndarray) -> bytes:
    return np.packbits(bits, bitorder="little").tobytes()


def window_bytes(spec: SourceSpec, bit_start: int, nbits: int) -> bytes:
    """Stream bits [bit_start, bit_start+nbits) as LSB-first bytes (iid kinds only;
    bit_start and nbits must be multiples of the sample width, and of 8 for b=1
    unless the caller re-aligns)."""
    b = spec.bits_per_sample
    if bit_start % b or nbits % b:
        raise ValueError("window must be sample aligned")
    vals = _samples_iid(spec, bit_start // b, nbits // b)
    if b == 1:
        return _pack_bits_host(vals)
    if b == 8:
        return vals.tobytes()
    raise ValueError("host windows support b in {1, 8}")


def stream_bytes_host(spec: SourceSpec, samples: int, chunk: int = 1 << 24) -> np.ndarray:
    """Whole stream on the host (uint8 array), generated in chunks.

    Chunked draws equal one-shot draws for PCG64, so this equals the reference's
    ``generate`` output for the same model and count.
    """
    b = spec.bits_per_sample
    nbytes = (samples * b + 7) // 8
    out = np.empty(nbytes, dtype=np.uint8)
    if spec.kind == "block-markov":
        return _block_markov_host(spec, samples)
    rng = np.random.default_rng(spec.seed)
    if b == 1:
        if chunk % 8:
            raise ValueError("chunk must be a multiple of 8 for bit streams")
        pos = 0
        for s in range(0, samples, chunk):
            c = min(chunk, samples - s)
            bits = (rng.random(c) < spec.p).astype(np.uint8)
            packed = np.packbits(bits, bitorder="little")
            out[pos:pos + packed.size] = packed
            pos += packed.size
        return out
    if b == 8:
        pmf = spec.pmf()
        for s in range(0, samples, chunk):
            c = min(chunk, samples - s)
            out[s:s + c] = rng.choice(len(pmf), size=c, p=pmf)
        return out
    raise ValueError("host streams support b in {1, 8}")


SPLITMIX_GAMMA = 0x9E3779B97F4A7C15
SEED_MIX = 0xD1B54A32D192ED03


def splitmix_bits_host(seed: int, bit0: int, nbits: int, p: float) -> np.ndarray:
    """Host restatement of bx_bernoulli_bits (for tests and small streams):
    bit i = (splitmix64(seed*SEED_MIX + i) >> 11) < p * 2^53, as 0/1 uint8."""
    with np.errstate(over="ignore"):
        z = np.uint64((seed * SEED_MIX) & (2**64 - 1)) + np.arange(bit0, bit0 + nbits, dtype=np.uint64)
        z = z + np.uint64(SPLITMIX_GAMMA)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    t = p * 2.0**53
    thr = np.uint64(2**53) if t >= 2.0**53 else np.uint64(max(0, int(t)))
    return ((z >> np.uint64(11)) < thr).astype(np.uint8)


def _block_markov_host(spec: SourceSpec, samples: int) -> np.ndarray:
    """Block-Markov bit stream (config 4), host restatement of the device
    generator: one counter-based stream of bits (seeded SplitMix64); the first
    block's bits are Bernoulli(1/2), every later block's bits are
    Bernoulli(flip) masks, and block k = block k-1 XOR mask_k."""
    B = spec.block_bits
    if B % 64 or samples % B:
        raise ValueError("block-markov needs 64-bit-multiple blocks dividing the stream")
    nblocks = samples // B
    first = splitmix_bits_host(spec.seed, 0, B, 0.5)
    rest = splitmix_bits_host(spec.seed, B, samples - B, spec.p)
    bits = np.concatenate([first, rest])
    words = np.packbits(bits, bitorder="little").view(np.uint64).reshape(nblocks, B // 64)
    return np.bitwise_xor.accumulate(words, axis=0).reshape(-1).view(np.uint8)


def _block_markov_device(spec: SourceSpec, samples: int, device=None):
    from . import device as D

    B = spec.block_bits
    if B % 64 or samples % B:
        raise ValueError("block-markov needs 64-bit-multiple blocks dividing the stream")
    dev = D.require_cuda(device)
    nbytes = samples // 8
    out = D.empty_stream(nbytes, dev)
    D.bernoulli_bits(B, 0.5, spec.seed, bit0=0, out=out)
    D.bernoulli_bits(samples - B, spec.p, spec.seed, bit0=B, out=out, out_byte0=B // 8)
    D.xor_scan_rows(out, samples // B, B // 8)
    return out, nbytes


# ---------------------------------------------------------------- device RNG

def to_model(spec: SourceSpec):
    from . import sources as S

    if spec.kind == "iid-biased":
        return S.iid_biased(spec.p, seed=spec.seed)
    if spec.kind == "iid-table":
        return S.iid_table(spec.pmf(), spec.bits_per_sample, seed=spec.seed)
    raise ValueError(f"no reference model for {spec.kind}")


def _draw_into(spec: SourceSpec, start: int, out: np.ndarray) -> None:
    """PCG64 doubles for samples [start, start+len(out)) of an iid stream,
    written in place (one 64-bit step per sample, reference sources.py:133-140)."""
    rng = np.random.default_rng(spec.seed)
    if start:
        rng.bit_generator.advance(start)
    rng.random(out.size, out=out)


def stream_range_device(spec: SourceSpec, start: int, count: int, device=None, *,
                        chunk: int = 1 << 22, threads: int | None = None):
    """Samples [start, start+count) of an iid stream as a packed, padded device
    buffer: ``(buffer, nbytes)``, byte-identical to the same slice of the
    reference ``generate`` output (sources.py:124-140).

    The PCG64 draws are the only host work; they are split into chunks drawn
    by ``threads`` host threads at once (each chunk from its own generator
    advanced to the chunk's first sample, numpy releases the GIL), straight
    into pinned buffers, while the device maps the previous wave of chunks to
    samples (threshold / inverse-CDF search, as numpy's ``choice`` does) and
    packs them (``bx_pack``).  This is how a rank of a sharded run generates
    only its own block range (sharding.shard_ranges).
    """
    import concurrent.futures as cf

    import torch

    from . import device as D

    if spec.kind not in ("iid-biased", "iid-table"):
        raise ValueError(f"range generation needs an iid kind, not {spec.kind}")
    b = spec.bits_per_sample
    if count < 1:
        raise ValueError("count must be >= 1")
    if (start * b) % 8:
        raise ValueError("range must start on a byte boundary of the stream")
    dev = D.require_cuda(device)
    nbytes = (count * b + 7) // 8
    out = D.empty_stream(nbytes, dev)
    out[(count * b // 32) * 4:].zero_()
    threads = threads or max(1, min(16, os.cpu_count() or 1))
    chunk = max(64, chunk // 64 * 64)         # whole words of output for b >= 1
    spans = [(s, min(chunk, count - s)) for s in range(0, count, chunk)]
    banks = [[torch.empty(chunk, dtype=torch.float64, pin_memory=True) for _ in range(threads)]
             for _ in range(2)]
    done = [None, None]
    stream = torch.cuda.Stream(dev)
    cdf_d = None
    if spec.kind == "iid-table":
        cdf = np.cumsum(spec.pmf())
        cdf /= cdf[-1]
        cdf_d = torch.from_numpy(cdf).to(dev)
    with cf.ThreadPoolExecutor(threads, thread_name_prefix="bx-draw") as pool, \
            torch.cuda.device(dev):
        for w in range(0, len(spans), threads):
            bank = banks[(w // threads) % 2]
            if done[(w // threads) % 2] is not None:
                done[(w // threads) % 2].synchronize()     # bank's previous H2D finished
            wave = spans[w:w + threads]
            list(pool.map(lambda a: _draw_into(spec, start + a[1][0], bank[a[0]][:a[1][1]].numpy()),
                          enumerate(wave)))
            with torch.cuda.stream(stream):
                for i, (s, c) in enumerate(wave):
                    u = bank[i][:c].to(dev, non_blocking=True)
                    if spec.kind == "iid-biased":
                        vals = (u < spec.p).to(torch.uint8)
                    else:
                        vals = torch.searchsorted(cdf_d, u, right=True).to(torch.uint8)
                    D.pack(vals, b, out=out, out_bit0=s * b, stream=stream)
                ev = torch.cuda.Event()
                ev.record(stream)
            done[(w // threads) % 2] = ev
        stream.synchronize()
    out.record_stream(stream)
    return out, nbytes


def stream_device(spec: SourceSpec, samples: int, device=None):
    """(padded device buffer, nbytes) of the stream; host PCG64 draws, device
    mapping and packing (byte-identical to ``stream_bytes_host``)."""
    from . import device as D
    from . import sources as S

    if spec.kind == "block-markov":
        return _block_markov_device(spec, samples, device)
    return S.generate_device(to_model(spec), samples, device)
