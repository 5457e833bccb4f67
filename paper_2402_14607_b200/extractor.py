"""Streaming two-source extraction with the reference's API, computed on B200.

Drop-in for ``blockext.extractor`` (reference pkg/src/blockext/extractor.py):
same names, parameters, output bit layout, report accounting and errors.  What
changes is where the work happens:

* framing, the GF(2^q) inner products and the output packing of every block
  run in one sm_100a kernel launch per segment (``bx_extract_eq``);
* the host keeps only the bookkeeping of the reference's ``BitReader``
  (bitio.py:25-64): it replays the exact sequence of ``read(size)`` calls the
  reference would make on each stream, in bulk, so ``*_bits_consumed``,
  ``*_discarded_tail_bits`` and the stop reason match bit for bit without a
  per-block Python loop.

Segments of up to ``segment_blocks`` blocks (a multiple of 64, so every segment
starts on a byte boundary of the inputs and of the output) bound host and
device memory on long or unbounded inputs.
"""
from __future__ import annotations

import io
import mmap
import os
import stat
import time
from dataclasses import dataclass
from typing import Iterable, Iterator, Sequence

import numpy as np

from . import params as _params
from .gf2q import MAX_FIELD_BITS, GFContext
from .params import error_bound_eq, error_bound_neq
from .report import ExtractionReport

READ_CHUNK = 1 << 16          # BitReader chunk size (reference bitio.py:25)
DEFAULT_SEGMENT_BLOCKS = 1 << 24
FIRST_LAZY_SEGMENT = 4096        # first chunks of an iteration arrive after 4096 blocks
ITER_PIECE = 1 << 16             # blocks unpacked at a time by __iter__ (multiple of 8)


@dataclass(frozen=True)
class OutputChunk:
    """One block's output: `width` bits, emitted in block order."""

    index: int   # 1-based block index
    bits: int
    width: int


@dataclass(frozen=True)
class BlockPair:
    """The paired input windows of one block, as field-element vectors."""

    index: int
    ctx: GFContext
    x: tuple[int, ...]
    y: tuple[int, ...]


@dataclass
class BlockCursor:
    """Streaming position: 1-based block and sample indices, current width."""

    block_index: int = 1
    sample_index: int = 1
    field_bits: int = 0

    def advance(self, vec_len: int, bits_per_sample: int, next_field_bits: int) -> None:
        self.sample_index += self.field_bits * vec_len // bits_per_sample
        self.block_index += 1
        self.field_bits = next_field_bits


class BlockProcessingError(RuntimeError):
    """A block failed; carries its 1-based index (reference extractor.py:69-74)."""

    def __init__(self, block_index: int, cause: BaseException):
        super().__init__(f"block {block_index} failed: {cause!r}")
        self.block_index = block_index


# ------------------------------------------------------------ device helpers

def _pack_vectors(vectors: Sequence[Sequence[int]], q: int) -> bytes:
    """Concatenate element vectors LSB-first into one q*n*len bit stream.

    Linear time: every element becomes ceil(q/8) little-endian bytes at a fixed
    stride, the (elements x q) bit matrix is cut out of them and re-packed in
    one ``packbits`` (no growing big-int shifts)."""
    flat = [v for vec in vectors for v in vec]
    if not flat:
        return b""
    nb = (q + 7) // 8
    if q % 8 == 0 and q <= 64:
        arr = np.array(flat, dtype=np.uint64).view(np.uint8).reshape(-1, 8)[:, :nb]
        return arr.tobytes()
    raw = np.frombuffer(b"".join(int(v).to_bytes(nb, "little") for v in flat),
                        dtype=np.uint8).reshape(-1, nb)
    bits = np.unpackbits(raw, axis=1, bitorder="little")[:, :q]
    return np.packbits(bits.reshape(-1), bitorder="little").tobytes()


def _unpack_fields(buf, count: int, q: int) -> list[int]:
    """The `count` consecutive q-bit fields at the start of the LSB-first bit
    string `buf`, as Python ints (linear time; inverse of ``_pack_vectors``)."""
    if count <= 0:
        return []
    a = np.frombuffer(buf, dtype=np.uint8, count=(count * q + 7) // 8)
    if q in (8, 16, 32, 64):
        return a.view(f"<u{q // 8}").tolist()
    bits = np.unpackbits(a, bitorder="little")[:count * q].reshape(count, q)
    width = 64 if q <= 64 else 128
    padded = np.zeros((count, width), dtype=np.uint8)
    padded[:, :q] = bits
    words = np.packbits(padded, axis=1, bitorder="little").view("<u8")
    if q <= 64:
        return words.reshape(-1).tolist()
    lo, hi = words[:, 0].tolist(), words[:, 1].tolist()
    return [a_ | (b_ << 64) for a_, b_ in zip(lo, hi)]


def _generic_inner_products(q: int, modulus: int, xs, ys, dev) -> list[int]:
    """Inner products under a caller-chosen modulus (bx_gf_ip_generic)."""
    import torch

    from . import _lib
    from . import device as D

    out = [0] * len(xs)
    groups: dict[int, list[int]] = {}
    for i, v in enumerate(xs):
        groups.setdefault(len(v), []).append(i)
    low = (modulus ^ (1 << q)).to_bytes(16, "little")
    mod_d = torch.frombuffer(bytearray(low), dtype=torch.uint8).to(dev)
    for n, idx in groups.items():
        xb = b"".join(int(v).to_bytes(16, "little") for i in idx for v in xs[i])
        yb = b"".join(int(v).to_bytes(16, "little") for i in idx for v in ys[i])
        xd = torch.frombuffer(bytearray(xb), dtype=torch.uint8).to(dev)
        yd = torch.frombuffer(bytearray(yb), dtype=torch.uint8).to(dev)
        res = torch.empty(16 * len(idx), dtype=torch.uint8, device=dev)
        with torch.cuda.device(dev):
            _lib.check(_lib.lib().bx_gf_ip_generic(q, mod_d.data_ptr(), xd.data_ptr(), yd.data_ptr(), n,
                                                   len(idx), res.data_ptr(), D.stream_ptr(None, dev)),
                       "bx_gf_ip_generic")
        host = res.cpu().numpy().tobytes()
        for k, i in enumerate(idx):
            out[i] = int.from_bytes(host[16 * k:16 * k + 16], "little")
    return out


def _device_inner_products(q: int, xs: Sequence[Sequence[int]], ys: Sequence[Sequence[int]],
                           device=None, modulus: int | None = None) -> list[int]:
    """sum_j x_j * y_j over GF(2^q) for each vector pair, on the GPU.

    Vectors are grouped by length; each group is one bx_extract_eq launch with
    one block per pair (default modulus), or one bx_gf_ip_generic launch for a
    caller-chosen modulus.  Elements must already be validated.
    """
    from . import device as D
    from .gf2q import modulus_int

    dev = D.require_cuda(device)
    if modulus is not None and modulus != modulus_int(q):
        return _generic_inner_products(q, modulus, xs, ys, dev)
    out = [0] * len(xs)
    groups: dict[int, list[int]] = {}
    for i, v in enumerate(xs):
        groups.setdefault(len(v), []).append(i)
    from . import sharding

    for n, idx in groups.items():
        xb = _pack_vectors([xs[i] for i in idx], q)
        yb = _pack_vectors([ys[i] for i in idx], q)
        # one C call (staging, H2D, kernel, D2H) for the usual small batch
        host = sharding.extract_small(xb, yb, q, n, len(idx), device=dev)
        if host is None:
            xd, xn = D.to_device_stream(xb, dev)
            yd, yn = D.to_device_stream(yb, dev)
            res = D.extract_eq(xd, xn, yd, yn, q, n, len(idx))
            nbytes = (len(idx) * q + 7) // 8
            host = res[:nbytes].cpu().numpy()
        for i, v in zip(idx, _unpack_fields(host.tobytes(), len(idx), q)):
            out[i] = v
    return out


def ext_ip(ctx: GFContext, x: Sequence[int], y: Sequence[int]) -> int:
    """Inner product sum(x_i * y_i) over GF(2^q) (reference extractor.py:77-87)."""
    if len(x) != len(y):
        raise ValueError(f"vector lengths differ: {len(x)} vs {len(y)}")
    if not x:
        raise ValueError("vectors must be non-empty")
    for v in x:
        ctx.check(v)
    for v in y:
        ctx.check(v)
    return _device_inner_products(ctx.q, [tuple(x)], [tuple(y)], modulus=ctx.modulus)[0]


def run_parallel(blocks: Iterable[BlockPair], workers: int, *,
                 capacity: int | None = None) -> Iterator[OutputChunk]:
    """Inner products of BlockPairs, in block order (reference extractor.py:94-130).

    Pairs are gathered into batches that grow 1, 2, 4, ... up to ``capacity``
    pairs (default 4096); each batch is one device launch per (q, n) group.  If
    the block source itself raises, the pairs already gathered are computed and
    yielded first (as the reference's lazy workers=1 loop would have), then the
    error propagates.  Output is identical for every
    ``workers`` value.  A pair with an out-of-range element raises ValueError at
    its position (workers == 1) or BlockProcessingError carrying its index
    (workers > 1), after all earlier chunks were yielded -- as the reference.
    """
    if workers < 1:
        raise ValueError("workers must be >= 1")
    batch_cap = capacity if capacity is not None else 4096
    batch_cap = max(1, batch_cap)
    it = iter(blocks)
    size = 1                 # batches grow 1, 2, 4, ... up to batch_cap, so a live
    while True:              # block source sees its first chunk after one pair
        batch: list[BlockPair] = []
        source_exc: BaseException | None = None
        try:
            for pair in it:
                batch.append(pair)
                if len(batch) >= size:
                    break
        except Exception as exc:  # noqa: BLE001 - the block source failed: flush, then re-raise
            source_exc = exc
        size = min(batch_cap, 2 * size)
        if not batch:
            if source_exc is not None:
                raise source_exc
            return
        bad_at = None
        bad_exc: Exception | None = None
        for k, pair in enumerate(batch):
            try:
                if len(pair.x) != len(pair.y):
                    raise ValueError(f"vector lengths differ: {len(pair.x)} vs {len(pair.y)}")
                if not pair.x:
                    raise ValueError("vectors must be non-empty")
                for v in pair.x:
                    pair.ctx.check(v)
                for v in pair.y:
                    pair.ctx.check(v)
            except Exception as exc:  # noqa: BLE001 - re-raised in order below
                bad_at, bad_exc = k, exc
                break
        good = batch if bad_at is None else batch[:bad_at]
        results = [0] * len(good)
        by_field: dict[tuple[int, int], list[int]] = {}
        for k, pair in enumerate(good):
            by_field.setdefault((pair.ctx.q, pair.ctx.modulus), []).append(k)
        for (q, mod), ks in by_field.items():
            vals = _device_inner_products(q, [good[k].x for k in ks], [good[k].y for k in ks],
                                          modulus=mod)
            for k, v in zip(ks, vals):
                results[k] = v
        for pair, v in zip(good, results):
            yield OutputChunk(pair.index, v, pair.ctx.q)
        if bad_exc is not None:
            if workers == 1:
                raise bad_exc
            raise BlockProcessingError(batch[bad_at].index, bad_exc) from bad_exc
        if source_exc is not None:
            raise source_exc


# ---------------------------------------------------------- stream sources

class _Source:
    """One input stream plus an exact replay of BitReader's bookkeeping.

    ``fill`` issues the same ``read(size)`` calls as reference bitio.py:35-43;
    ``take`` mirrors a successful ``read_bits`` (:45-60).  In-memory inputs
    (bytes, bytearray, memoryview, numpy arrays, torch tensors) are never
    copied by the replay; file-like inputs are read for real and their bytes
    are kept until the blocks that use them are computed.
    """

    def __init__(self, stream, allow_map: bool = True):
        self._mem = None
        self._file = None
        try:
            import torch
            is_tensor = isinstance(stream, torch.Tensor)
        except ImportError:  # pragma: no cover
            is_tensor = False
        if is_tensor:
            self._mem = stream.reshape(-1).view(__import__("torch").uint8)
            self._total = self._mem.numel()
        elif isinstance(stream, np.ndarray):
            self._mem = np.ascontiguousarray(stream).reshape(-1).view(np.uint8)
            self._total = self._mem.size
        elif isinstance(stream, (bytes, bytearray, memoryview)):
            self._mem = memoryview(stream).cast("B")
            self._total = len(self._mem)
        elif allow_map and self._map_file(stream):
            pass
        elif hasattr(stream, "read"):
            self._file = stream
            # delivered bytes live in one numpy buffer: [_start, _start + _len)
            # holds stream bytes [_parts_base, _parts_base + _len).  Standard
            # io readers fill it in place with readinto (same call sizes and
            # semantics as read(size)); other objects go through read().
            self._buf = None
            self._keep = None         # owner of _buf when it is a pinned tensor
            self._start = 0
            self._len = 0
            self._parts_base = 0
            self._readinto = isinstance(stream, (io.BufferedIOBase, io.RawIOBase)) and \
                hasattr(stream, "readinto")
            self._size_hint = self.known_bytes()
        else:
            raise TypeError(f"cannot read from {type(stream).__name__}")
        self.buffered = 0             # bytes delivered by read() so far
        self.consumed = 0             # bits handed out (BitReader.bits_consumed)
        self.exhausted = False

    #: regular files at least this large are memory-mapped (smaller ones are read)
    MAP_MIN_BYTES = 1 << 20

    def _map_file(self, stream) -> bool:
        """Regular binary files are mapped read-only (page cache, no read()
        copies) and replayed like in-memory bytes; reads of a regular file
        return min(size, remaining) bytes, so the closed-form BitReader replay
        holds, and the file's position is kept where the reference's read()
        calls would have left it (_sync_pos)."""
        if not isinstance(stream, (io.BufferedReader, io.FileIO)):
            return False
        self._pos_file = None
        try:
            fd = stream.fileno()
            st = os.fstat(fd)
            if not stat.S_ISREG(st.st_mode):
                return False
            pos = stream.tell()
            if st.st_size - pos < self.MAP_MIN_BYTES:
                return False
            flags = mmap.MAP_SHARED | getattr(mmap, "MAP_POPULATE", 0)
            self._map = mmap.mmap(fd, st.st_size, flags=flags, prot=mmap.PROT_READ)
        except (AttributeError, OSError, ValueError, io.UnsupportedOperation):
            return False
        self._mem = memoryview(self._map)[pos:]
        self._total = st.st_size - pos
        self._pos_file, self._pos0 = stream, pos
        return True

    def _sync_pos(self) -> None:
        if getattr(self, "_pos_file", None) is not None:
            self._pos_file.seek(self._pos0 + self.buffered)

    def avail(self) -> int:
        return self.buffered * 8 - self.consumed

    def known_bytes(self) -> int | None:
        """Bytes this stream can still deliver, when knowable without reading
        (in-memory inputs; regular files); None for pipes and sockets."""
        if self._mem is not None:
            return self._total - self.buffered
        try:
            st = os.fstat(self._file.fileno())
            if not stat.S_ISREG(st.st_mode):
                return None
            return max(0, st.st_size - self._file.tell())
        except (AttributeError, OSError, ValueError, io.UnsupportedOperation):
            return None

    #: largest buffer allocated up front from a regular file's size; beyond it
    #: the buffer grows geometrically (consumed bytes are released per segment)
    PREALLOC_MAX = 1 << 30

    def _reserve(self, need: int) -> None:
        """Room for `need` more bytes after the held ones (amortised O(1):
        compaction or geometric growth, never a copy per read)."""
        cap = 0 if self._buf is None else self._buf.size
        end = self._start + self._len
        if end + need <= cap:
            return
        if self._len + need <= cap and self._start >= self._len:
            # compact: the released prefix is at least as large as the live data
            self._buf[:self._len] = self._buf[self._start:end]
            self._start = 0
            return
        first = self._size_hint if (self._buf is None and self._size_hint) else 0
        new_cap = max(self._len + need, 2 * cap, min(first, self.PREALLOC_MAX), 1 << 20)
        buf, keep = self._host_buffer(new_cap)
        if self._len:
            buf[:self._len] = self._buf[self._start:end]
        self._buf, self._keep, self._start = buf, keep, 0

    @staticmethod
    def _host_buffer(nbytes: int):
        """Pinned host memory when CUDA is up (pre-faulted, reused through
        torch's host allocator cache, and the chunks' H2D then goes straight
        from it without staging copies); plain numpy memory otherwise."""
        try:
            import torch
            if torch.cuda.is_available():
                t = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
                return t.numpy(), t
        except (ImportError, RuntimeError):  # pragma: no cover - no CUDA runtime
            pass
        return np.empty(nbytes, dtype=np.uint8), None

    def _read(self, need: int) -> int:
        if self._mem is not None:
            got = min(need, self._total - self.buffered)
            return max(got, 0)
        self._reserve(need)
        end = self._start + self._len
        if self._readinto:
            got = self._file.readinto(memoryview(self._buf)[end:end + need]) or 0
        else:
            data = self._file.read(need)
            got = len(data) if data else 0
            if got:
                self._buf[end:end + got] = np.frombuffer(data, dtype=np.uint8)
        self._len += got
        return got

    def fill(self, want_bits: int) -> None:
        while self.avail() < want_bits and not self.exhausted:
            need = max(READ_CHUNK, (want_bits - self.avail() + 7) // 8)
            got = self._read(need)
            if got == 0:
                self.exhausted = True
                break
            self.buffered += got
        self._sync_pos()

    def take(self, nbits: int) -> bool:
        """read_bits(nbits): False (nothing consumed) if fewer bits remain."""
        self.fill(nbits)
        if self.avail() < nbits:
            return False
        self.consumed += nbits
        return True

    def tail_bits(self) -> int:
        return self.avail()

    def bulk_capacity(self, B: int) -> int | None:
        """Blocks of B bits this in-memory source can still serve, or None if the
        closed form does not apply (file-like source, or blocks > one read)."""
        if self._mem is None or B > 8 * READ_CHUNK:
            return None
        return (8 * self._total - self.consumed) // B

    def bulk_take(self, B: int, k: int) -> None:
        """Consume k blocks at once.  Valid when bulk_capacity(B) >= k: with
        blocks no larger than one 64 KiB read, every refill is exactly one read
        of READ_CHUNK bytes, so after T consumed bits BitReader has made
        ceil(T / (8*READ_CHUNK)) reads (bitio.py:35-43)."""
        self.consumed += k * B
        reads = -(-self.consumed // (8 * READ_CHUNK))
        self.buffered = max(self.buffered, min(self._total, reads * READ_CHUNK))
        self._sync_pos()

    def window(self, byte_lo: int, byte_hi: int):
        """Stream bytes [byte_lo, byte_hi) (all already delivered)."""
        if self._mem is not None:
            return self._mem[byte_lo:byte_hi]
        lo = self._start + byte_lo - self._parts_base
        return memoryview(self._buf)[lo:lo + byte_hi - byte_lo]

    def release(self, byte_lo: int) -> None:
        """Forget buffered file bytes before stream offset byte_lo."""
        if self._file is not None and byte_lo > self._parts_base:
            cut = min(byte_lo - self._parts_base, self._len)
            self._start += cut
            self._len -= cut
            self._parts_base += cut


# ------------------------------------------------------------- extraction

class Extraction:
    """One extraction run: iterate for chunks or call ``run``; then read ``.report``.

    Single-use, like the reference (extractor.py:133-279).  Extra keyword
    arguments (not in the reference): ``device`` (CUDA device for the kernels),
    ``devices`` (a list of devices to shard each segment's blocks across) and
    ``segment_blocks`` (blocks computed per launch).
    """

    def __init__(self, x_stream, y_stream, plan, *, workers: int = 1,
                 max_blocks: int | None = None, device=None, devices=None,
                 segment_blocks: int = DEFAULT_SEGMENT_BLOCKS):
        # one file object feeding both streams is read alternately (x, y, x,
        # ...) exactly as the reference does; only distinct objects are mapped
        shared = x_stream is y_stream
        self._x = _Source(x_stream, allow_map=not shared)
        self._y = _Source(y_stream, allow_map=not shared)
        self.plan = plan
        self.mode = "eq" if _params.is_eq_plan(plan) else "neq"
        self._workers = workers
        self._max_blocks = max_blocks
        self._device = device
        self._devices = list(devices) if devices else None
        self._segment = max(64, (int(segment_blocks) // 64) * 64)
        self._lazy = False               # __iter__: grow segments from FIRST_LAZY_SEGMENT
        self._out_buf = None             # run(sink): whole-run pinned output (eq mode)
        self._out_pos = 0
        self._started = False
        self._used_bits = 0
        self._stop_reason = "completed"
        self._chunks_emitted = 0
        self._output_bits = 0
        self._widths: list[int] = []     # neq: width of every completed block
        self._t0 = 0.0
        self.cursor = BlockCursor(field_bits=self._first_width())
        self.report: ExtractionReport | None = None

    # -- plan helpers (reference extractor.py:165-180)
    def _first_width(self) -> int:
        return self.plan.field_bits if self.mode == "eq" else self.plan.first_field_bits

    def _next_width(self, width: int) -> int:
        if self.mode == "eq":
            return width
        return width + self.plan.growth * self.plan.bits_per_sample

    def _block_limit(self) -> int | None:
        if self.mode == "eq":
            if self._max_blocks is None:
                return self.plan.num_blocks
            return min(self.plan.num_blocks, self._max_blocks)
        return self._max_blocks

    # -- bookkeeping replay
    def _advance(self, width: int, n: int, count_cap: int | None) -> int:
        """Consume up to count_cap blocks of `width`; returns how many completed.

        Sets ``_stop_reason`` to "input-exhausted" when a stream runs dry.
        """
        B = width * n
        x, y = self._x, self._y
        done = 0
        cx, cy = x.bulk_capacity(B), y.bulk_capacity(B)
        if cx is not None and cy is not None:
            k = min(cx, cy) if count_cap is None else min(cx, cy, count_cap)
            if k > 0:
                x.bulk_take(B, k)
                y.bulk_take(B, k)
                done = k
        while count_cap is None or done < count_cap:
            k = min(x.avail() // B, y.avail() // B)
            if count_cap is not None:
                k = min(k, count_cap - done)
            if k > 0:
                x.consumed += k * B
                y.consumed += k * B
                done += k
                continue
            okx = x.take(B)      # both reads always happen (extractor.py:194-195)
            oky = y.take(B)
            if not (okx and oky):
                self._stop_reason = "input-exhausted"
                break
            done += 1
        self._used_bits += done * B
        return done

    # -- device compute of a run of equal-width blocks
    def _compute(self, width: int, n: int, count: int, bit: int) -> bytes:
        """Packed output bytes of `count` blocks whose windows start at stream
        bit `bit` of both inputs; the last byte is zero-padded."""
        from . import sharding

        B = width * n
        lo, hi = bit // 8, (bit + count * B + 7) // 8
        out = None
        if self._out_buf is not None:
            # run(sink), eq mode: D2H straight into the run's single output
            # buffer (segments are multiples of 64 blocks, so every segment but
            # the last ends on a byte boundary)
            out = self._out_buf[self._out_pos:]
            self._out_pos += (count * width) // 8
        return sharding.extract_packed(self._x.window(lo, hi), self._y.window(lo, hi), width, n,
                                       count, x_bit0=bit % 8, y_bit0=bit % 8,
                                       device=self._device, devices=self._devices, out=out)

    def _segments_eq(self) -> Iterator[tuple[int, int, bytes]]:
        """Yield (first_block, count, packed_output) segment by segment
        (block loop of reference extractor.py:182-208)."""
        plan = self.plan
        width, n = plan.field_bits, plan.vec_len
        if width > MAX_FIELD_BITS:
            self._stop_reason = "width-cap"
            return
        limit = self._block_limit()
        B = width * n
        done = 0
        while done < limit:
            cap = min(self._seg_cap(done), limit - done)
            got = self._advance(width, n, cap)
            if got:
                out = self._compute(width, n, got, done * B)
                self._x.release((done + got) * B // 8)
                self._y.release((done + got) * B // 8)
                yield done, got, out
            done += got
            if got < cap:
                return
        self._stop_reason = "completed" if limit == plan.num_blocks else "block-limit"

    def _segments_neq(self) -> Iterator[tuple[int, int, bytes]]:
        """Incremental widths q_k = q1 + (k-1)*growth*b (extractor.py:170-173).

        growth = 0 runs in bulk segments like eq mode; growth >= 1 stops at the
        128-bit width cap after <= 128 blocks, so the bookkeeping replays block by
        block and the device computes all blocks in one bx_extract_neq call."""
        plan = self.plan
        n = plan.vec_len
        limit = self._block_limit()
        step = plan.growth * plan.bits_per_sample
        width = plan.first_field_bits
        if step == 0:
            done = 0
            offset = 0
            while limit is None or done < limit:
                if width > MAX_FIELD_BITS:
                    self._stop_reason = "width-cap"
                    return
                seg = self._seg_cap(done)
                cap = seg if limit is None else min(seg, limit - done)
                got = self._advance(width, n, cap)
                if got:
                    out = self._compute(width, n, got, offset)
                    self._widths.extend([width] * got)
                    offset += got * width * n
                    self._x.release(offset // 8)
                    self._y.release(offset // 8)
                    yield done, got, out
                    done += got
                if got < cap:
                    return
            self._stop_reason = "block-limit"
            return
        done = 0
        stopped = False
        while limit is None or done < limit:
            if width > MAX_FIELD_BITS:
                self._stop_reason = "width-cap"
                stopped = True
                break
            if self._advance(width, n, 1) == 0:
                stopped = True
                break
            self._widths.append(width)
            done += 1
            width += step
        if not stopped:
            self._stop_reason = "block-limit"
        if done:
            from . import sharding

            total_in = (self._used_bits + 7) // 8
            out = sharding.extract_neq_packed(self._x.window(0, total_in), self._y.window(0, total_in),
                                              plan.first_field_bits, step, n, done,
                                              device=self._device)
            yield 0, done, out

    # -- public protocol
    def _begin(self) -> None:
        if self._started:
            raise RuntimeError("an Extraction is single-use; create a new one")
        self._started = True
        self._t0 = time.perf_counter()
        if self._workers < 1:
            raise ValueError("workers must be >= 1")

    #: largest single output buffer run(sink) preallocates (pinned host memory)
    OUT_BUF_MAX = 4 << 30

    def _alloc_out_buf(self) -> None:
        """eq mode, more than one segment: one pinned buffer for the whole
        output, so segments D2H into place and the sink gets one zero-copy
        write (instead of joining per-segment buffers)."""
        if self.mode != "eq" or self.plan.field_bits > MAX_FIELD_BITS:
            return
        width, B = self.plan.field_bits, self.plan.field_bits * self.plan.vec_len
        blocks = self._block_limit()
        for src in (self._x, self._y):
            kb = src.known_bytes()
            if kb is not None:
                blocks = min(blocks, (8 * kb + src.avail()) // B)
        if blocks <= self._segment:
            return                      # one segment: its own buffer is already whole
        nbytes = (blocks * width + 7) // 8
        if nbytes > self.OUT_BUF_MAX:
            return
        import torch

        self._out_buf = torch.empty(nbytes + 1, dtype=torch.uint8,
                                    pin_memory=torch.cuda.is_available())
        self._out_pos = 0

    def _seg_cap(self, done: int) -> int:
        """Blocks in the next segment.  ``run`` uses full segments; iteration
        starts at FIRST_LAZY_SEGMENT blocks and doubles, so the first chunks of
        a live stream come out quickly and long runs still use big launches."""
        if not self._lazy:
            return self._segment
        grown = FIRST_LAZY_SEGMENT
        while grown <= done and grown < self._segment:
            grown *= 2
        return min(grown, self._segment)

    def _segments(self) -> Iterator[tuple[int, int, bytes]]:
        return self._segments_eq() if self.mode == "eq" else self._segments_neq()

    def __iter__(self) -> Iterator[OutputChunk]:
        self._lazy = True
        try:
            self._begin()
        except ValueError:
            self._finalize()
            raise
        try:
            for first, count, packed in self._segments():
                widths = ([self.plan.field_bits] * count if self.mode == "eq"
                          else self._widths[first:first + count])
                buf = np.frombuffer(memoryview(packed), dtype=np.uint8) \
                    if not isinstance(packed, np.ndarray) else packed.reshape(-1).view(np.uint8)
                if widths and widths[0] == widths[-1] and len(set(widths)) == 1:
                    # constant width: unpack ITER_PIECE blocks at a time (pieces
                    # start on byte boundaries), linear in the segment length
                    w = widths[0]
                    for p0 in range(0, count, ITER_PIECE):
                        c = min(ITER_PIECE, count - p0)
                        lo = p0 * w // 8
                        vals = _unpack_fields(buf[lo:lo + (c * w + 7) // 8], c, w)
                        for k, bits in enumerate(vals):
                            self._chunks_emitted += 1
                            self._output_bits += w
                            yield OutputChunk(first + p0 + k + 1, bits, w)
                    continue
                # growing widths (neq, <= 128 blocks before the width cap)
                val = int.from_bytes(buf.tobytes(), "little")
                for k, w in enumerate(widths):
                    bits = val & ((1 << w) - 1)
                    val >>= w
                    self._chunks_emitted += 1
                    self._output_bits += w
                    yield OutputChunk(first + k + 1, bits, w)
        finally:
            self._finalize()

    def run(self, sink=None) -> ExtractionReport:
        """Consume the run; optionally write the packed output to `sink` (one write)."""
        try:
            self._begin()
        except ValueError:
            self._finalize()
            raise
        parts: list[bytes] = []
        carry = 0          # neq: bit-level concatenation of variable-width segments
        carry_bits = 0
        if sink is not None:
            self._alloc_out_buf()
        try:
            for first, count, packed in self._segments():
                if self.mode == "eq":
                    nbits = count * self.plan.field_bits
                else:
                    nbits = sum(self._widths[first:first + count])
                self._chunks_emitted += count
                self._output_bits += nbits
                if sink is None or self._out_buf is not None:
                    continue
                if carry_bits == 0 and nbits % 8 == 0:
                    parts.append(packed)
                else:
                    carry |= int.from_bytes(bytes(packed), "little") << carry_bits
                    carry_bits += nbits
                    whole = carry_bits // 8
                    if whole:
                        parts.append((carry & ((1 << (8 * whole)) - 1)).to_bytes(whole, "little"))
                        carry >>= 8 * whole
                        carry_bits -= 8 * whole
        finally:
            self._finalize()
        if sink is not None and self._out_buf is not None:
            nbytes = (self._output_bits + 7) // 8
            sink.write(memoryview(self._out_buf.numpy()[:nbytes]))
            self._out_buf = None
            self.report.pad_bits = (-self._output_bits) % 8
        elif sink is not None:
            if carry_bits:
                parts.append(carry.to_bytes(1, "little"))
            if len(parts) == 1:
                sink.write(memoryview(parts[0]))
            else:
                sink.write(b"".join(bytes(p) for p in parts))
            self.report.pad_bits = (-self._output_bits) % 8
        return self.report

    def _finalize(self) -> None:
        if self.report is not None:
            return
        wall = time.perf_counter() - self._t0
        k = self._chunks_emitted
        exhausted = self._stop_reason == "input-exhausted"
        if self.mode == "eq":
            bound = error_bound_eq(self.plan, k)
        else:
            bound = error_bound_neq(self.plan, k) if k else float("-inf")
        # cursor: one advance per completed block (extractor.py:205)
        n, b = self.plan.vec_len, self.plan.bits_per_sample
        if self.mode == "eq" or self.plan.growth == 0:
            w = self._first_width()       # constant width: closed form of k advances
            self.cursor.sample_index += k * (w * n // b)
            self.cursor.block_index += k
        else:
            for w in self._widths[:k]:
                self.cursor.advance(n, b, self._next_width(w))
        self.report = ExtractionReport(
            mode=self.mode,
            plan=self.plan,
            blocks_completed=k,
            x_bits_consumed=self._x.consumed,
            y_bits_consumed=self._y.consumed,
            output_bits=self._output_bits,
            x_discarded_tail_bits=self._discarded(self._x, exhausted),
            y_discarded_tail_bits=self._discarded(self._y, exhausted),
            log2_error_bound=bound,
            wall_time_s=wall,
            window_disjointness=True,
            stop_reason=self._stop_reason,
        )

    def _discarded(self, src: _Source, exhausted: bool) -> int:
        # reference extractor.py:249-262
        d = src.consumed - self._used_bits
        if exhausted:
            d += src.tail_bits()
        elif self._stop_reason == "completed" and self.mode == "eq":
            d += self.plan.num_samples * self.plan.bits_per_sample - self._used_bits
        return d


def extract_eq(x_stream, y_stream, plan, *, workers: int = 1, max_blocks: int | None = None,
               **kw) -> Extraction:
    """Equal-block extraction (reference extractor.py:282-291)."""
    if not _params.is_eq_plan(plan):
        raise TypeError("extract_eq needs an EqPlan")
    return Extraction(x_stream, y_stream, plan, workers=workers, max_blocks=max_blocks, **kw)


def extract_neq(x_stream, y_stream, plan, *, workers: int = 1, max_blocks: int | None = None,
                **kw) -> Extraction:
    """Incremental-block extraction (reference extractor.py:294-306)."""
    if not _params.is_neq_plan(plan) or _params.is_eq_plan(plan):
        raise TypeError("extract_neq needs a NeqPlan")
    return Extraction(x_stream, y_stream, plan, workers=workers, max_blocks=max_blocks, **kw)


__all__ = ["BlockCursor", "BlockPair", "BlockProcessingError", "Extraction", "OutputChunk",
           "ext_ip", "extract_eq", "extract_neq", "run_parallel"]
