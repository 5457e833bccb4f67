"""Block-range sharding across GPUs.

Blocks are independent (reference extractor.py:16-19; isolation pinned by
pkg/tests/test_extractor.py:125-137), so a run of `count` blocks splits into
contiguous ranges, one per device, with no collective: each device gets its
own input window, computes its blocks, and its packed output lands at a fixed
byte offset of the result.  Range starts are multiples of 64 blocks, so every
range's input starts on a byte boundary (64*q*n bits) and its output on a
64*q-bit (byte) boundary.

Two entry points:
* ``extract_packed`` -- one process, several devices (threads, one per device);
* ``rank_range``     -- the per-rank slice for torch.distributed launches
  (bench.py), where each rank owns one GPU.
"""
from __future__ import annotations

import os
import threading

import numpy as np

ALIGN_BLOCKS = 64


def shard_ranges(nblocks: int, parts: int, align: int = ALIGN_BLOCKS) -> list[tuple[int, int]]:
    """Split [0, nblocks) into `parts` contiguous (start, count) ranges whose
    starts are multiples of `align`; trailing ranges may be empty."""
    if parts < 1:
        raise ValueError("parts must be >= 1")
    units = -(-nblocks // align)
    base, extra = divmod(units, parts)
    out = []
    start = 0
    for p in range(parts):
        u = base + (1 if p < extra else 0)
        cnt = min(u * align, nblocks - start) if start < nblocks else 0
        out.append((start, max(cnt, 0)))
        start += u * align
    return out


def rank_range(nblocks: int, rank: int, world: int) -> tuple[int, int]:
    return shard_ranges(nblocks, world)[rank]


def _slice(buf, lo: int, hi: int):
    return buf[lo:hi]


# host->device pipeline granularity per stream (BX_PIPE_MB overrides)
PIPE_CHUNK_BYTES = int(os.environ.get("BX_PIPE_MB", "64")) << 20


def _as_tensor(buf):
    """Zero-copy torch view of a host buffer (bytes-like / numpy) or the tensor."""
    import torch

    if isinstance(buf, torch.Tensor):
        return buf.reshape(-1).view(torch.uint8)
    arr = np.frombuffer(memoryview(buf), dtype=np.uint8) if not isinstance(buf, np.ndarray) \
        else np.ascontiguousarray(buf).reshape(-1).view(np.uint8)
    import warnings
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        return torch.from_numpy(arr)


def _device_view(t, nbytes: int, dev):
    """Use a device tensor in place when it lives on `dev`, is 16-byte aligned
    and its storage holds the ABI's guard bytes (round_up(n, 16) + 16);
    otherwise copy it into a padded buffer (one device-to-device pass)."""
    from . import device as D

    tail = t.untyped_storage().nbytes() - t.storage_offset() * t.element_size()
    if (t.device == dev and t.data_ptr() % 16 == 0 and t.is_contiguous()
            and tail >= D.padded_len(nbytes)):
        return t
    buf, _ = D.to_device_stream(t[:nbytes], dev)
    return buf


class _Stager:
    """Run-ahead staging of one pageable operand: a producer thread copies
    chunk k into a free slot of a pinned ring (the copy is split over worker
    threads; numpy copies release the GIL), enqueues the slot's H2D on the
    operand's copy stream and hands the compute loop a CUDA event for it.  A
    slot is refilled only after its previous H2D completed (event), so the
    producer runs up to SLOTS - 1 chunks ahead of the transfers.  x and y each
    get their own producer, so the two host copies and the two H2D streams all
    overlap.  The path is host-memory bound: a staged byte costs a host read,
    a host write and a DMA read (copy alone 56 GB/s on 8 threads,
    tools/host_copy_bw.py); 128 MiB chunks reach ~300 Gbit/s raw input on
    config 2 against ~240 with 64 MiB (fewer fill/drain phases)."""

    SLOTS = 3
    THREADS = int(os.environ.get("BX_STAGE_THREADS", "8"))

    _pool = None
    _pool_lock = threading.Lock()

    @classmethod
    def pool(cls):
        """Process-wide copy workers (shared by every device's stagers)."""
        with cls._pool_lock:
            if cls._pool is None:
                import concurrent.futures as cf

                cls._pool = cf.ThreadPoolExecutor(cls.THREADS, thread_name_prefix="bx-stage")
            return cls._pool

    def __init__(self, slot_bytes: int, dev, stream, slots: int):
        import queue

        import torch

        self.slot_bytes = slot_bytes
        self._dev, self._stream = dev, stream
        self._slots = max(1, min(self.SLOTS, slots))
        self._bufs = [torch.empty(slot_bytes, dtype=torch.uint8, pin_memory=True)
                      for _ in range(self._slots)]
        self._done = [None] * self._slots
        self._q: queue.Queue = queue.Queue()
        self._t = None

    def start(self, chunks) -> None:
        """chunks: list of (host source tensor, device destination tensor)."""
        self._t = threading.Thread(target=self._run, args=(chunks,), daemon=True)
        self._t.start()

    def _run(self, chunks) -> None:
        import torch

        try:
            with torch.cuda.device(self._dev):
                parts_max = max(1, self.THREADS // 2)
                pool = self.pool()
                for k, (src, dst) in enumerate(chunks):
                    s = k % self._slots
                    if self._done[s] is not None:
                        self._done[s].synchronize()
                    n = src.numel()
                    if n > self.slot_bytes:
                        raise ValueError("chunk larger than a staging slot")
                    hs, hb = src.numpy(), self._bufs[s][:n].numpy()
                    parts = max(1, min(parts_max, n >> 22))
                    edges = [n * i // parts for i in range(parts + 1)]
                    list(pool.map(
                        lambda i: np.copyto(hb[edges[i]:edges[i + 1]], hs[edges[i]:edges[i + 1]]),
                        range(parts)))
                    with torch.cuda.stream(self._stream):
                        dst.copy_(self._bufs[s][:n], non_blocking=True)
                        ev = torch.cuda.Event()
                        ev.record(self._stream)
                    self._done[s] = ev
                    self._q.put(ev)
        except BaseException as exc:  # noqa: BLE001 - re-raised by next()
            self._q.put(exc)

    def next(self):
        """CUDA event of the next chunk's H2D (raises the producer's error)."""
        item = self._q.get()
        if isinstance(item, BaseException):
            raise item
        return item

    def close(self) -> None:
        if self._t is not None:
            self._t.join()
        for ev in self._done:
            if ev is not None:
                ev.synchronize()


#: host inputs up to this many bytes (x + y) take the one-shot small path
SMALL_INPUT_BYTES = int(os.environ.get("BX_SMALL_MB", "16")) << 20


class _SmallPath:
    """Per-device cached buffers for short host runs (the real-time case: one
    call per capture chunk).  Both windows are copied into one pinned staging
    buffer at 16-byte aligned, zero-padded offsets, cross in ONE H2D, compute,
    and the packed output comes back in one D2H -- no stream creation, no
    staging threads, no per-call device allocation (the
    fixed cost of extract_eq(...).run() on config 1)."""

    _by_dev: dict = {}
    _lock = threading.Lock()

    def __init__(self, dev):
        self.dev = dev
        self.lock = threading.Lock()
        self.host = None      # pinned uint8 staging
        self.devbuf = None    # device uint8: x | y | out

    @classmethod
    def get(cls, dev) -> "_SmallPath":
        with cls._lock:
            sp = cls._by_dev.get(dev.index)
            if sp is None:
                sp = cls._by_dev[dev.index] = cls(dev)
            return sp

    def run(self, xt, yt, xn: int, yn: int, q: int, n: int, count: int, x_bit0: int,
            y_bit0: int, out, out_byte0: int, res=None, rbit: int = 0) -> None:
        import torch

        from . import device as D

        px, py = D.padded_len(xn), D.padded_len(yn)
        obytes = (count * q + 7) // 8
        po = D.padded_len(obytes)
        with self.lock:
            if self.host is None or self.host.numel() < px + py:
                self.host = torch.empty(max(px + py, 1 << 20), dtype=torch.uint8, pin_memory=True)
            if self.devbuf is None or self.devbuf.numel() < px + py + po:
                self.devbuf = torch.empty(max(px + py + po, 1 << 20), dtype=torch.uint8,
                                          device=self.dev)
            st = torch.cuda.current_stream(self.dev)
            d = self.devbuf
            if xt.is_pinned() and yt.is_pinned():
                d[:xn].copy_(xt[:xn], non_blocking=True)
                d[px:px + yn].copy_(yt[:yn], non_blocking=True)
                d[xn:px].zero_()
                d[px + yn:px + py].zero_()
            else:
                h = self.host.numpy()
                h[:xn] = xt[:xn].numpy()
                h[xn:px] = 0
                h[px:px + yn] = yt[:yn].numpy()
                h[px + yn:px + py] = 0
                d[:px + py].copy_(self.host[:px + py], non_blocking=True)
            xd, yd = d[:px], d[px:px + py]
            if res is None:
                res, rbit = d[px + py:px + py + po], 0
                res.zero_()
            D.extract_eq(xd, xn, yd, yn, q, n, count, x_bit0=x_bit0, y_bit0=y_bit0, out=res,
                         out_bit0=rbit, stream=st)
            if out is not None:
                out[out_byte0:out_byte0 + obytes].copy_(res[:obytes], non_blocking=True)
            st.synchronize()   # staging and device buffers are reused by the next call


_STREAMS: dict = {}
_STREAMS_LOCK = threading.Lock()


def _copy_streams(dev):
    """(x copy, y copy, output copy) streams of a device, created once per
    process (stream creation costs tens of microseconds per call)."""
    import torch

    with _STREAMS_LOCK:
        st = _STREAMS.get(dev.index)
        if st is None:
            st = _STREAMS[dev.index] = tuple(torch.cuda.Stream(dev) for _ in range(3))
        return st


def _extract_one_device(xv, yv, q: int, n: int, count: int, x_bit0: int, y_bit0: int, dev,
                        out, out_byte0: int, dev_out=None) -> None:
    """`count` blocks on one device.  Host inputs are streamed in ~64 MiB chunks
    on a copy stream while earlier chunks compute (one launch per chunk); device
    inputs are used in place (copied once if they lack the guard padding).
    The packed output goes to host `out` at byte out_byte0 (D2H), or, with
    ``dev_out = (tensor, bit0)``, straight from the kernels into that device
    buffer (which may live on a peer GPU: NVLink stores, no D2H)."""
    import torch

    from . import device as D

    if count <= 0:
        return
    B = q * n
    xt, yt = _as_tensor(xv), _as_tensor(yv)
    xn, yn = (x_bit0 + count * B + 7) // 8, (y_bit0 + count * B + 7) // 8
    obytes = (count * q + 7) // 8
    if not (xt.is_cuda or yt.is_cuda) and xn + yn <= SMALL_INPUT_BYTES:
        if dev_out is None and xt.is_contiguous() and yt.is_contiguous():
            # one C call: staging, H2D, kernel, D2H, synchronise
            from . import _lib
            _lib.check(_lib.lib().bx_extract_eq_host(
                xt.data_ptr(), xt.numel(), x_bit0, yt.data_ptr(), yt.numel(), y_bit0, q, n, count,
                out.data_ptr() + out_byte0, dev.index), "bx_extract_eq_host")
            return
        res, rbit = dev_out if dev_out is not None else (None, 0)
        with torch.cuda.device(dev):
            _SmallPath.get(dev).run(xt, yt, xn, yn, q, n, count, x_bit0, y_bit0,
                                    None if dev_out is not None else out, out_byte0, res, rbit)
        return
    with torch.cuda.device(dev):
        comp = torch.cuda.current_stream(dev)
        if dev_out is None:
            res, rbit = torch.zeros(D.padded_len(obytes), dtype=torch.uint8, device=dev), 0
        else:
            res, rbit = dev_out
        co = None
        if xt.is_cuda and yt.is_cuda:
            xd = _device_view(xt, xn, dev)
            yd = _device_view(yt, yn, dev)
            D.extract_eq(xd, xn, yd, yn, q, n, count, x_bit0=x_bit0, y_bit0=y_bit0, out=res,
                         out_bit0=rbit)
        else:
            xd = D.empty_stream(xn, dev)
            yd = D.empty_stream(yn, dev)
            pinned = xt.is_pinned() and yt.is_pinned()
            # x and y chunks travel on two copy streams (two DMA engines) while
            # the compute stream runs each chunk as soon as both halves landed;
            # pageable inputs are first staged through pinned rings by run-ahead
            # host threads (see _Stager) so their H2D is asynchronous too
            cx, cy, co_cached = _copy_streams(dev)
            # each chunk's output words go back on their own stream as soon as
            # the chunk's kernel finished (D2H overlaps the next chunks' H2D:
            # PCIe is full duplex); chunk boundaries sit on multiples of 64
            # blocks, i.e. on whole output words, so chunks never share a word
            co = co_cached if dev_out is None and out.is_pinned() else None
            slot = int(os.environ.get("BX_STAGE_MB", "128")) << 20
            step = max(ALIGN_BLOCKS, (PIPE_CHUNK_BYTES * 8 // B) // ALIGN_BLOCKS * ALIGN_BLOCKS)
            if not pinned:
                step = max(ALIGN_BLOCKS, (slot * 8 // B - 16) // ALIGN_BLOCKS * ALIGN_BLOCKS)
            spans = []
            done = 0
            while done < count:
                cnt = min(step, count - done)
                xs, ys = x_bit0 + done * B, y_bit0 + done * B
                spans.append((done, cnt, xs, ys, xs // 8, (xs + cnt * B + 7) // 8,
                              ys // 8, (ys + cnt * B + 7) // 8))
                done += cnt
            stagers = []
            try:
                if not pinned:
                    # ring slots sized to the largest chunk (small runs pin little)
                    slot = max(max(sp[5] - sp[4], sp[7] - sp[6]) for sp in spans)
                    stagers = [_Stager(slot, dev, cx, len(spans)), _Stager(slot, dev, cy, len(spans))]
                    stagers[0].start([(xt[sp[4]:sp[5]], xd[sp[4]:sp[5]]) for sp in spans])
                    stagers[1].start([(yt[sp[6]:sp[7]], yd[sp[6]:sp[7]]) for sp in spans])
                for done, cnt, xs, ys, xlo, xhi, ylo, yhi in spans:
                    if pinned:
                        with torch.cuda.stream(cx):
                            xd[xlo:xhi].copy_(xt[xlo:xhi], non_blocking=True)
                        with torch.cuda.stream(cy):
                            yd[ylo:yhi].copy_(yt[ylo:yhi], non_blocking=True)
                        comp.wait_stream(cx)
                        comp.wait_stream(cy)
                    else:
                        comp.wait_event(stagers[0].next())
                        comp.wait_event(stagers[1].next())
                    D.extract_eq(xd, xn, yd, yn, q, n, cnt, x_bit0=xs, y_bit0=ys, out=res,
                                 out_bit0=rbit + done * q, stream=comp)
                    if co is not None:
                        olo, ohi = done * q // 8, ((done + cnt) * q + 7) // 8
                        co.wait_stream(comp)
                        with torch.cuda.stream(co):
                            out[out_byte0 + olo:out_byte0 + ohi].copy_(res[olo:ohi], non_blocking=True)
            finally:
                for st in stagers:
                    st.close()
            xd.record_stream(cx)
            yd.record_stream(cy)
            if co is not None:
                res.record_stream(co)
                co.synchronize()
        if dev_out is None and co is None:
            # D2H straight into this range of the (pinned) result
            out[out_byte0:out_byte0 + obytes].copy_(res[:obytes], non_blocking=True)
        comp.synchronize()


def extract_neq_packed(xv, yv, q1: int, step: int, n: int, count: int, *, device=None) -> bytes:
    """Packed output of `count` incremental-width blocks (widths q1 + k*step)
    read from bit 0 of xv / yv: one H2D of the consumed prefix, one
    bx_extract_neq call, one D2H."""
    import torch

    from . import device as D

    dev = D.require_cuda(device)
    total_in = sum((q1 + k * step) * n for k in range(count))
    total_out = sum(q1 + k * step for k in range(count))
    nb = (total_in + 7) // 8
    with torch.cuda.device(dev):
        xd, xn = D.to_device_stream(_as_tensor(xv)[:nb], dev)
        yd, yn = D.to_device_stream(_as_tensor(yv)[:nb], dev)
        res = D.extract_neq(xd, xn, yd, yn, q1, step, n, count)
        return res[:(total_out + 7) // 8].cpu().numpy().tobytes()


def _host_array(buf):
    """Zero-copy uint8 numpy view of a host buffer (None for CUDA tensors)."""
    if isinstance(buf, np.ndarray):
        return np.ascontiguousarray(buf).reshape(-1).view(np.uint8)
    if isinstance(buf, (bytes, bytearray, memoryview)):
        return np.frombuffer(memoryview(buf).cast("B"), dtype=np.uint8)
    try:
        import torch
        if isinstance(buf, torch.Tensor) and not buf.is_cuda:
            return buf.reshape(-1).view(torch.uint8).numpy()
    except ImportError:  # pragma: no cover
        pass
    return None


def extract_small(xv, yv, q: int, n: int, count: int, *, x_bit0: int = 0, y_bit0: int = 0,
                  device=None):
    """Packed output of a short run from host memory through one C call
    (bx_extract_eq_host), or None when the inputs are not plain host buffers
    or the run is too large for the one-shot path."""
    from . import _lib
    from . import device as D

    xa, ya = _host_array(xv), _host_array(yv)
    if xa is None or ya is None:
        return None
    B = q * n
    xn, yn = (x_bit0 + count * B + 7) // 8, (y_bit0 + count * B + 7) // 8
    if xn + yn > SMALL_INPUT_BYTES or xa.size < xn or ya.size < yn:
        return None
    dev = D.require_cuda(device)
    out = np.empty((count * q + 7) // 8, dtype=np.uint8)
    _lib.check(_lib.lib().bx_extract_eq_host(xa.ctypes.data, xa.size, x_bit0, ya.ctypes.data,
                                             ya.size, y_bit0, q, n, count, out.ctypes.data,
                                             dev.index), "bx_extract_eq_host")
    return out


def extract_packed(xv, yv, q: int, n: int, count: int, *, x_bit0: int = 0, y_bit0: int = 0,
                   device=None, devices=None, out=None) -> np.ndarray:
    """Packed output of `count` blocks (uint8 array over pinned memory; the last
    byte is zero-padded); xv/yv hold the windows (host buffers or
    torch tensors) starting at bit x_bit0 / y_bit0 of their first byte.  With
    several devices the blocks are split into contiguous 64-aligned ranges, one
    per device, each driven by its own host thread.  `out` (a CPU uint8 tensor
    of at least ceil(count*q/8) bytes, ideally pinned) receives the bytes
    instead of a fresh pinned buffer."""
    from . import device as D

    if out is None and not (devices and len(devices) > 1):
        # short host runs: one C call (bx_extract_eq_host), no torch orchestration
        small = extract_small(xv, yv, q, n, count, x_bit0=x_bit0, y_bit0=y_bit0,
                              device=devices[0] if devices else device)
        if small is not None:
            return small

    import torch

    devs = [D.require_cuda(d) for d in devices] if devices else [D.require_cuda(device)]
    B = q * n
    obytes = (count * q + 7) // 8
    if out is None:
        # small host runs come back through bx_extract_eq_host's own pinned
        # staging (a memcpy), so their result needs no pinned allocation
        small = len(devs) == 1 and 2 * ((x_bit0 + count * B + 7) // 8) <= SMALL_INPUT_BYTES
        out = torch.empty(obytes, dtype=torch.uint8, pin_memory=not small)
    else:
        out = out[:obytes]
    ranges = [r for r in shard_ranges(count, len(devs)) if r[1] > 0]
    errors: list[BaseException] = []

    def work(dev, start: int, cnt: int) -> None:
        try:
            xs, ys = x_bit0 + start * B, y_bit0 + start * B
            _extract_one_device(_slice(xv, xs // 8, (xs + cnt * B + 7) // 8),
                                _slice(yv, ys // 8, (ys + cnt * B + 7) // 8),
                                q, n, cnt, xs % 8, ys % 8, dev, out, start * q // 8)
        except BaseException as exc:  # noqa: BLE001 - re-raised on the caller's thread
            errors.append(exc)

    if len(ranges) <= 1:
        for dev, (s, c) in zip(devs, ranges):
            work(dev, s, c)
    else:
        ts = [threading.Thread(target=work, args=(d, s, c)) for d, (s, c) in zip(devs, ranges)]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
    if errors:
        raise errors[0]
    return out.numpy()       # a view of the pinned buffer (kept alive by the array)


def distributed_extract(xv, yv, q: int, n: int, count: int, *, x_bit0: int = 0,
                        y_bit0: int = 0, group=None, compute=None, device=None,
                        gather: str = "object", to_host: bool = True,
                        local_input: bool = False):
    """Multi-process form (one process per GPU, torch.distributed).

    Every rank sees the same run (e.g. a shared capture file or a shared seeded
    generator) and computes only its contiguous block range ``rank_range``;
    rank 0 returns the whole packed output (other ranks return None).  There is
    no collective on the input path; only outputs (1/(2n) of the input bytes)
    move, in one of two ways:

    * ``gather="object"``: each rank's packed part (host bytes) is gathered to
      rank 0 through the process group (any backend; ``compute`` lets CPU
      tests inject a stand-in for the GPU step);
    * ``gather="peer"``: rank 0 allocates the output in its HBM and shares it
      over CUDA IPC; every rank's extraction kernels store their range of it
      directly -- peer stores over NVLink from the kernel epilogue, so the
      gather is fused into the compute and no extra collective or copy runs.
      Ranges start at multiples of 64 blocks (64*q bits = whole 32-bit words),
      so ranks never share an output word.  Rank 0 returns host bytes, or the
      device tensor with ``to_host=False``.  Requires every process to see
      rank 0's GPU under the same index (torchrun's default visibility).
    """
    if gather == "peer":
        return _distributed_extract_peer(xv, yv, q, n, count, x_bit0=x_bit0, y_bit0=y_bit0,
                                         group=group, device=device, to_host=to_host,
                                         local_input=local_input)
    if gather != "object":
        raise ValueError(f"unknown gather mode {gather!r}")
    import torch.distributed as dist

    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    start, cnt = rank_range(count, rank, world)
    B = q * n
    part = b""
    if cnt:
        xs, ys = (x_bit0, y_bit0) if local_input else (x_bit0 + start * B, y_bit0 + start * B)
        fn = compute or (lambda *a, **k: extract_packed(*a, device=device, **k))
        part = fn(xv[xs // 8:(xs + cnt * B + 7) // 8], yv[ys // 8:(ys + cnt * B + 7) // 8],
                  q, n, cnt, x_bit0=xs % 8, y_bit0=ys % 8)
    parts = [None] * world if rank == 0 else None
    dist.gather_object((start, cnt, part), parts, dst=0, group=group)
    if rank != 0:
        return None
    out = bytearray((count * q + 7) // 8)
    for s, c, p in parts:
        if c:
            ob = s * q // 8
            out[ob:ob + len(p)] = p
    return bytes(out)


def _distributed_extract_peer(xv, yv, q: int, n: int, count: int, *, x_bit0: int, y_bit0: int,
                              group, device, to_host: bool, local_input: bool = False):
    """gather="peer" of :func:`distributed_extract`."""
    import torch
    import torch.distributed as dist
    from torch.multiprocessing.reductions import reduce_tensor

    from . import device as D

    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    dev = D.require_cuda(device)
    obytes = (count * q + 7) // 8
    if rank == 0:
        buf = torch.zeros(D.padded_len(obytes), dtype=torch.uint8, device=dev)
        torch.cuda.synchronize(dev)       # zeroed before any peer stores into it
        shared = [reduce_tensor(buf)]
    else:
        shared = [None]
    dist.broadcast_object_list(shared, src=0, group=group)
    if rank != 0:
        rebuild, args = shared[0]
        buf = rebuild(*args)              # rank 0's buffer mapped into this process
    start, cnt = rank_range(count, rank, world)
    B = q * n
    failure = None
    try:
        if cnt:
            xs, ys = (x_bit0, y_bit0) if local_input else (x_bit0 + start * B, y_bit0 + start * B)
            _extract_one_device(_slice(xv, xs // 8, (xs + cnt * B + 7) // 8),
                                _slice(yv, ys // 8, (ys + cnt * B + 7) // 8),
                                q, n, cnt, xs % 8, ys % 8, dev, None, 0,
                                dev_out=(buf, start * q))
        torch.cuda.synchronize(dev)
    except Exception as exc:  # noqa: BLE001 - re-raised after the barrier protocol
        failure = exc
    # the barriers run on every rank whatever happened above, so a failing
    # rank cannot leave the others waiting in a collective; every rank then
    # learns whether any range failed
    dist.barrier(group=group)           # every range is in rank 0's buffer
    flag = torch.tensor([0 if failure is None else 1], dtype=torch.int32,
                        device=dev if dist.get_backend(group) == "nccl" else "cpu")
    dist.all_reduce(flag, group=group)
    if rank != 0:
        del buf
        dist.barrier(group=group)       # rank 0 may free the buffer after this
        if failure is not None:
            raise failure
        if int(flag.item()):
            raise RuntimeError("distributed_extract: another rank's range failed")
        return None
    dist.barrier(group=group)
    if failure is not None:
        raise failure
    if int(flag.item()):
        raise RuntimeError("distributed_extract: another rank's range failed")
    res = buf[:obytes]
    return res.cpu().numpy().tobytes() if to_host else res
