"""GPU parity: the sm_100a kernels through the public API vs the reference's
recorded outputs (tests/golden) and vs the CPU oracle.  Bit-exact throughout."""
import io
import random

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import paper_2402_14607_b200 as bx
from paper_2402_14607_b200 import _lib, device as D
from oracle import coracle

from bxtest_util import DribbleIO, case_inputs, report_dict, tiny_eq_plan

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def need_cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    _lib.lib()


def dev_run(xb, yb, q, n, k, x_bit0=0, y_bit0=0, out_bit0=0, prefill=None):
    xd, xn = D.to_device_stream(xb, "cuda")
    yd, yn = D.to_device_stream(yb, "cuda")
    nbytes = (out_bit0 + k * q + 7) // 8
    out = torch.zeros(D.padded_len(nbytes), dtype=torch.uint8, device="cuda")
    if prefill is not None:
        out[:nbytes] = torch.from_numpy(np.frombuffer(prefill, dtype=np.uint8)[:nbytes]).cuda()
    D.extract_eq(xd, xn, yd, yn, q, n, k, x_bit0=x_bit0, y_bit0=y_bit0, out=out, out_bit0=out_bit0)
    return out[:nbytes].cpu().numpy().tobytes()


def test_eq_cases_through_api(golden):
    for c in golden("eq_cases.json"):
        xb, yb = case_inputs(c)
        plan = tiny_eq_plan(bx, c["b"], c["samples"], c.get("rate", "3/4"), c["n"], c["q"])
        sink = io.BytesIO()
        rep = bx.extract_eq(xb, yb, plan, max_blocks=c.get("max_blocks")).run(sink)
        assert sink.getvalue().hex() == c["out"], c["tag"]
        assert report_dict(rep) == c["report"], c["tag"]


def test_neq_cases_through_api(golden):
    for c in golden("neq_cases.json"):
        if c.get("zeros"):
            xb = yb = bytes(c["x_len"])
        else:
            xb, yb = case_inputs(c)
        plan = bx.plan_neq(c["b"], "3/4", c["q1"], c["growth"])
        sink = io.BytesIO()
        rep = bx.extract_neq(xb, yb, plan, max_blocks=c["max_blocks"]).run(sink)
        assert sink.getvalue().hex() == c["out"]
        assert report_dict(rep) == c["report"]


def test_every_q_random_shapes_and_offsets():
    rnd = random.Random(1234)
    for q in range(1, 129):
        for _ in range(3):
            n = rnd.choice([1, 2, 3, rnd.randint(1, 40), rnd.randint(40, 300)])
            k = rnd.randint(1, 700)
            xo, yo = rnd.randint(0, 70), rnd.randint(0, 70)
            oo = rnd.choice([0, rnd.randint(1, 100)])
            nb = (max(xo, yo) + k * q * n + 7) // 8 + rnd.randint(0, 9)
            xb, yb = rnd.randbytes(nb), rnd.randbytes(nb)
            want = coracle.extract_eq(xb, yb, q, n, k, x_bit0=xo, y_bit0=yo)
            got = dev_run(xb, yb, q, n, k, x_bit0=xo, y_bit0=yo, out_bit0=oo,
                          prefill=bytes([0xA5]) * ((oo + k * q + 7) // 8))
            gi = int.from_bytes(got, "little")
            assert (gi >> oo) & ((1 << (k * q)) - 1) == int.from_bytes(want, "little"), (q, n, k, xo, yo, oo)
            # bits outside the written range are preserved
            pre = int.from_bytes(bytes([0xA5]) * len(got), "little")
            keep = ((1 << len(got) * 8) - 1) ^ (((1 << (k * q)) - 1) << oo)
            assert gi & keep == pre & keep


def test_extremes_all_ones_and_zeros():
    # 24, 40, 48, 56: the period kernel; 58, 80: the planner / paper TMA shapes
    for q in (1, 2, 4, 7, 8, 9, 16, 24, 31, 32, 33, 40, 48, 56, 58, 63, 64, 65, 80, 100, 127, 128):
        for n in (1, 5, 48, 64, 257):
            k = 40
            nb = (k * q * n + 7) // 8
            for fill in (b"\xff", b"\x00", b"\x55"):
                xb = fill * nb
                yb = b"\xff" * nb
                assert dev_run(xb, yb, q, n, k) == coracle.extract_eq(xb, yb, q, n, k), (q, n, fill)


def test_gf_mul_kats(golden):
    for q in range(1, 129):
        rows = golden("gf_mul.json")[str(q)]
        a = [int(r[0], 16) for r in rows]
        b = [int(r[1], 16) for r in rows]
        assert bx.field(q).mul_many(a, b) == [int(r[2], 16) for r in rows], q
    assert bx.gf_mul(bx.field(2), 0b10, 0b10) == 0b11


def test_ext_ip_kats(golden):
    for c in golden("ext_ip.json"):
        ctx = bx.field(c["q"])
        xs = [int(v, 16) for v in c["x"]]
        ys = [int(v, 16) for v in c["y"]]
        assert bx.ext_ip(ctx, xs, ys) == int(c["z"], 16)
    with pytest.raises(ValueError):
        bx.ext_ip(bx.field(2), (1,), (1, 2))
    with pytest.raises(ValueError):
        bx.ext_ip(bx.field(2), (), ())
    with pytest.raises(ValueError):
        bx.ext_ip(bx.field(2), (4,), (1,))


def test_field_inverses_small():
    for q in range(1, 9):
        ctx = bx.field(q)
        xs = [x for x in range(1, 1 << q) for _ in range(1, 1 << q)]
        ys = [y for _ in range(1, 1 << q) for y in range(1, 1 << q)]
        prods = ctx.mul_many(xs, ys)
        for x in range(1, 1 << q):
            row = prods[(x - 1) * ((1 << q) - 1):x * ((1 << q) - 1)]
            assert row.count(1) == 1          # exactly one inverse
            assert len(set(row)) == (1 << q) - 1  # multiplication by x is a bijection


def test_field_pow_and_inv_one_launch():
    """GFContext.pow / inv (reference gf2q.py:171-189) as one bx_gf_pow launch,
    against square-and-multiply over the oracle's field product; exponents
    beyond 128 bits, e = 0, x = 0, the default and a custom modulus."""
    from oracle import pyoracle
    from paper_2402_14607_b200 import _lib
    rnd = random.Random(77)

    def ref_pow(q, mod, x, e):
        r = 1
        while e:
            if e & 1:
                r = pyoracle.gf_mul(q, mod, r, x)
            x = pyoracle.gf_mul(q, mod, x, x)
            e >>= 1
        return r

    for q in (1, 2, 7, 8, 16, 31, 32, 63, 64, 80, 127, 128):
        ctx = bx.field(q)
        xs = [0, 1] + [rnd.getrandbits(q) for _ in range(6)]
        es = [0, 5] + [rnd.getrandbits(rnd.choice([3, 40, 130, 300])) for _ in range(6)]
        for x, e in zip(xs, es):
            e_ref = e if (e < (1 << q) - 1 or x == 0) else e % ((1 << q) - 1)
            if x == 0 and e > 0:
                want = 0
            else:
                want = ref_pow(q, ctx.modulus, x, e_ref)
            assert ctx.pow(x, e) == want, (q, x, e)
        n0 = _lib.launch_count()
        x = rnd.getrandbits(q) | 1
        inv = ctx.inv(x)
        assert _lib.launch_count() - n0 == 1          # one device launch per inverse
        assert ctx.mul(x, inv) == 1
    with pytest.raises(ZeroDivisionError):
        bx.field(8).inv(0)
    with pytest.raises(ValueError):
        bx.field(8).pow(3, -1)
    # a non-default irreducible modulus: x^8 + x^4 + x^3 + x + 1 (AES)
    ctx = bx.GFContext(8, 0x11B)
    for x in range(1, 256):
        assert pyoracle.gf_mul(8, 0x11B, x, ctx.inv(x)) == 1


def test_run_parallel_order_and_errors():
    ctx = bx.field(4)
    rnd = random.Random(14)
    pairs = [bx.BlockPair(i + 1, ctx, tuple(rnd.randrange(16) for _ in range(3)),
                          tuple(rnd.randrange(16) for _ in range(3))) for i in range(4)]
    chunks = list(bx.run_parallel(iter(pairs), workers=4))
    assert [c.index for c in chunks] == [1, 2, 3, 4]
    assert [c.bits for c in chunks] == [bx.ext_ip(ctx, p.x, p.y) for p in pairs]
    good = bx.BlockPair(1, ctx, (1, 2), (3, 4))
    bad = bx.BlockPair(2, ctx, (1, 99), (3, 4))
    with pytest.raises(bx.BlockProcessingError) as ei:
        list(bx.run_parallel(iter([good, bad]), workers=2))
    assert ei.value.block_index == 2
    with pytest.raises(ValueError):
        list(bx.run_parallel(iter([good, bad]), workers=1))


def test_c1_full(golden):
    from paper_2402_14607_b200 import workloads as W
    wl = W.WORKLOADS["c1"]
    xb = W.stream_bytes_host(wl.x, wl.samples).tobytes()
    yb = W.stream_bytes_host(wl.y, wl.samples).tobytes()
    sink = io.BytesIO()
    rep = bx.extract_eq(xb, yb, wl.plan()).run(sink)
    assert sink.getvalue() == golden("c1_out.bin")
    assert report_dict(rep) == golden("c1.json")["report"]


def test_streams_dribble_and_chunk_invariance():
    rnd = random.Random(3)
    data_x, data_y = rnd.randbytes(500), rnd.randbytes(500)
    plan = tiny_eq_plan(bx, 8, 500, "3/4", 5, 8)
    whole = [c.bits for c in bx.extract_eq(data_x, data_y, plan)]
    dribble = [c.bits for c in bx.extract_eq(DribbleIO(data_x, 1), DribbleIO(data_y, 1), plan)]
    assert whole == dribble and len(whole) == plan.num_blocks


def test_block_isolation():
    rnd = random.Random(4)
    plan = tiny_eq_plan(bx, 8, 120, "3/4", 6, 8)
    base_x = bytearray(rnd.randbytes(120))
    data_y = rnd.randbytes(120)
    base = [c.bits for c in bx.extract_eq(bytes(base_x), data_y, plan)]
    for target in (0, 7, 19):
        m = bytearray(base_x)
        bit = target * 48 + rnd.randrange(48)
        m[bit // 8] ^= 1 << (bit % 8)
        got = [c.bits for c in bx.extract_eq(bytes(m), data_y, plan)]
        assert [i for i, (a, b) in enumerate(zip(base, got)) if a != b] == [target]


def test_device_tensor_inputs_and_segments():
    rnd = random.Random(21)
    q, n, k = 56, 48, 5000
    nb = k * q * n // 8
    xb, yb = rnd.randbytes(nb), rnd.randbytes(nb)
    plan = tiny_eq_plan(bx, 8, nb, "3/4", n, q)
    want = coracle.extract_eq(xb, yb, q, n, k)
    xt = torch.frombuffer(bytearray(xb), dtype=torch.uint8).cuda()
    yt = torch.frombuffer(bytearray(yb), dtype=torch.uint8).cuda()
    # padded device tensors are used in place (zero-copy path)
    xp = torch.zeros(nb + 64, dtype=torch.uint8, device="cuda")
    yp = torch.zeros(nb + 64, dtype=torch.uint8, device="cuda")
    xp[:nb] = xt
    yp[:nb] = yt
    for src in ((xb, yb), (xt, yt), (xp[:nb], yp[:nb])):
        for seg in (64, 1000, 1 << 24):
            sink = io.BytesIO()
            bx.extract_eq(*src, plan, segment_blocks=seg).run(sink)
            assert sink.getvalue() == want


def test_host_pipeline_chunking(monkeypatch):
    """Host inputs stream through the chunked H2D pipeline: pageable inputs via
    the run-ahead pinned rings (many chunks, ring wrap-around), pinned inputs
    via the two copy streams, each chunk's output D2H on its own stream; every
    chunking gives the oracle's bytes, at byte-aligned and odd bit offsets."""
    rnd = random.Random(22)
    q, n = 56, 48
    k = 3 * 64 * 40 + 17                     # ~2.7 MB per stream, a ragged last chunk
    for lead in (0, 3):                      # odd start bits: x_bit0 = y_bit0 = lead
        nb = (lead + k * q * n + 7) // 8
        xb, yb = rnd.randbytes(nb), rnd.randbytes(nb)
        want = coracle.extract_eq(xb, yb, q, n, k, x_bit0=lead, y_bit0=lead)
        from paper_2402_14607_b200 import sharding
        for mb in ("1", "128"):
            monkeypatch.setenv("BX_STAGE_MB", mb)
            got = sharding.extract_packed(xb, yb, q, n, k, x_bit0=lead, y_bit0=lead)
            assert got.tobytes()[:len(want)] == want, ("pageable", mb, lead)
        monkeypatch.setattr(sharding, "PIPE_CHUNK_BYTES", 1 << 20)
        xt = torch.frombuffer(bytearray(xb), dtype=torch.uint8).pin_memory()
        yt = torch.frombuffer(bytearray(yb), dtype=torch.uint8).pin_memory()
        got = sharding.extract_packed(xt, yt, q, n, k, x_bit0=lead, y_bit0=lead)
        assert got.tobytes()[:len(want)] == want, ("pinned", lead)
        monkeypatch.setattr(sharding, "PIPE_CHUNK_BYTES", 64 << 20)


def test_mapped_file_inputs(tmp_path):
    """Regular files >= 1 MiB take the memory-mapped path: output equals the
    oracle, and with max_blocks the files stop where the reference's 64 KiB
    reads would leave them (as BytesIO sources of the same bytes do)."""
    rnd = random.Random(23)
    q, n = 56, 48
    k = 4000                                  # 1.34 MB per stream (>= the 1 MiB map threshold)
    nb = k * q * n // 8 + 5000
    xb, yb = rnd.randbytes(nb), rnd.randbytes(nb)
    (tmp_path / "x").write_bytes(xb)
    (tmp_path / "y").write_bytes(yb)
    plan = tiny_eq_plan(bx, 8, nb, "3/4", n, q)
    full = plan.num_blocks
    want = coracle.extract_eq(xb, yb, q, n, full)
    for limit in (None, 777):
        with open(tmp_path / "x", "rb") as fx, open(tmp_path / "y", "rb") as fy:
            run = bx.extract_eq(fx, fy, plan, max_blocks=limit)
            assert run._x._pos_file is fx
            sink = io.BytesIO()
            rep = run.run(sink)
            m = full if limit is None else limit
            got = int.from_bytes(sink.getvalue(), "little")
            assert got == int.from_bytes(want, "little") & ((1 << (m * q)) - 1)
            bxio, byio = io.BytesIO(xb), io.BytesIO(yb)
            rep2 = bx.extract_eq(bxio, byio, plan, max_blocks=limit).run(io.BytesIO())
            assert report_dict(rep) == report_dict(rep2)
            assert (fx.tell(), fy.tell()) == (bxio.tell(), byio.tell())


def test_pack_kats(golden):
    for c in golden("pack.json"):
        vals = np.array([int(v, 16) for v in c["values"]], dtype=np.uint64)
        t = torch.from_numpy(vals.view(np.int64)).cuda()
        out = D.pack(t, c["b"])
        nbytes = len(c["out"]) // 2
        assert out[:nbytes].cpu().numpy().tobytes().hex() == c["out"], c["b"]


def test_pack_random_offsets_and_widths():
    rnd = random.Random(8)
    for elem, dt in ((1, torch.uint8), (2, torch.int16), (4, torch.int32), (8, torch.int64)):
        for _ in range(12):
            b = rnd.randint(1, 8 * elem)
            cnt = rnd.randint(1, 3000)
            off = rnd.randint(0, 77)
            vals = [rnd.getrandbits(8 * elem) for _ in range(cnt)]
            arr = np.array(vals, dtype=np.dtype(f"u{elem}"))
            t = torch.from_numpy(arr.view(np.dtype(f"i{elem}"))).cuda()
            want = coracle.pack([v & ((1 << b) - 1) for v in vals], b)
            out = D.pack(t, b, out_bit0=off)
            got = int.from_bytes(out.cpu().numpy().tobytes(), "little") >> off
            assert got & ((1 << (cnt * b)) - 1) == int.from_bytes(want, "little")


def test_output_canaries_and_giant_blocks():
    """Writes stay inside [out_bit0, out_bit0 + k*q) even at buffer ends, and
    blocks too large for shared memory (direct global reads) are exact."""
    rnd = random.Random(99)
    for q, n, k, xo in [(64, 20000, 3, 5), (128, 9000, 2, 0), (7, 100_000, 2, 3), (33, 1, 5000, 1),
                        (4, 64, 1, 0), (128, 8, 1, 0)]:
        nb = (xo + k * q * n + 7) // 8
        xb, yb = rnd.randbytes(nb), rnd.randbytes(nb)
        want = int.from_bytes(coracle.extract_eq(xb, yb, q, n, k, x_bit0=xo, y_bit0=xo), "little")
        xd, xn = D.to_device_stream(xb, "cuda")
        yd, yn = D.to_device_stream(yb, "cuda")
        for oo in (0, 13):
            obytes = (oo + k * q + 7) // 8
            buf = torch.full((obytes + 64,), 0x5A, dtype=torch.uint8, device="cuda")
            view = buf[:D.padded_len(obytes)]
            D.extract_eq(xd, xn, yd, yn, q, n, k, x_bit0=xo, y_bit0=xo, out=view, out_bit0=oo)
            host = buf.cpu().numpy().tobytes()
            gi = int.from_bytes(host[:obytes], "little")
            assert (gi >> oo) & ((1 << (k * q)) - 1) == want, (q, n, k, oo)
            pre = int.from_bytes(bytes([0x5A]) * obytes, "little")
            keep = ((1 << obytes * 8) - 1) ^ (((1 << (k * q)) - 1) << oo)
            assert gi & keep == pre & keep
            assert host[obytes:] == bytes([0x5A]) * 64, "write past the output range"


def test_bitio_pack_values_round_trip():
    from paper_2402_14607_b200.bitio import pack_values, unpack_values
    rnd = random.Random(12)
    for width in (1, 3, 11, 33, 64, 80, 128):
        vals = [rnd.getrandbits(width) for _ in range(57)]
        data, pad = pack_values(vals, width)
        assert len(data) * 8 == width * len(vals) + pad
        assert unpack_values(data, width, len(vals)) == vals
        assert data == coracle.pack(vals, width)


def test_lazy_iteration_matches_run():
    """Iteration uses growing segments (4096, 8192, ...); chunks must equal run()."""
    rnd = random.Random(31)
    q, n, k = 13, 5, 20_000
    nb = (k * q * n + 7) // 8
    xb, yb = rnd.randbytes(nb), rnd.randbytes(nb)
    plan = tiny_eq_plan(bx, 1, k * q * n, "3/4", n, q)
    chunks = list(bx.extract_eq(xb, yb, plan))
    assert len(chunks) == k and [c.index for c in chunks[:2]] == [1, 2]
    acc = 0
    for i, c in enumerate(chunks):
        acc |= c.bits << (i * q)
    sink = io.BytesIO()
    bx.extract_eq(xb, yb, plan).run(sink)
    assert acc.to_bytes(len(sink.getvalue()), "little") == sink.getvalue()
    assert sink.getvalue() == coracle.extract_eq(xb, yb, q, n, k)


@pytest.mark.parametrize("depth", [1, 2, 3])
def test_native_pipe_random_push_sizes(depth):
    """bx_pipe: any sequence of push sizes equals one run over the concatenation,
    synchronous (depth 1) and with 1-2 pushes in flight."""
    from paper_2402_14607_b200.pipe import Pipe
    rnd = random.Random(17 + depth)
    for q, n in [(4, 64), (13, 7), (56, 48), (128, 8), (1, 3), (80, 71)]:
        total = rnd.randint(20_000, 120_000)
        xb, yb = rnd.randbytes(total), rnd.randbytes(total)
        out = []
        with Pipe(q, n, chunk_bytes=9000, depth=depth) as p:
            pos = 0
            while pos < total:
                step = min(total - pos, rnd.choice([1, 7, 100, 4096, 9000]))
                out.append(p.push(xb[pos:pos + step], yb[pos:pos + step]))
                pos += step
            out.append(p.flush())
            k = p.blocks
        assert k == total * 8 // (q * n)
        assert b"".join(out) == coracle.extract_eq(xb, yb, q, n, k), (q, n)


def test_tma_tiles_of_one_width_interleaved():
    """One kernel width launched with tiles of different shared-memory sizes
    in turn (large, smaller, large again): the kernel's dynamic shared-memory
    limit must never be lowered under a memoised larger configuration."""
    rnd = random.Random(123)
    for q in (72, 80, 99):
        for n in (200, 61, 200, 33, 150, 200):
            k = 40
            nb = (k * q * n + 7) // 8 + 16
            xb, yb = rnd.randbytes(nb), rnd.randbytes(nb)
            xd, xn = D.to_device_stream(xb, "cuda")
            yd, yn = D.to_device_stream(yb, "cuda")
            got = D.extract_eq(xd, xn, yd, yn, q, n, k, x_bit0=3, y_bit0=3)
            want = coracle.extract_eq(xb, yb, q, n, k, x_bit0=3, y_bit0=3)
            assert got[:len(want)].cpu().numpy().tobytes() == want, (q, n)


def test_native_pipe_async_latency_and_errors():
    """depth 2: a push returns the previous push's output; capacity and
    in-flight misuse are reported through bx_last_error."""
    import ctypes

    from paper_2402_14607_b200 import _lib
    from paper_2402_14607_b200.pipe import Pipe
    q, n = 16, 64
    B = q * n // 8
    rnd = random.Random(5)
    xb, yb = rnd.randbytes(8 * B), rnd.randbytes(8 * B)
    want = coracle.extract_eq(xb, yb, q, n, 8)
    with Pipe(q, n, chunk_bytes=4 * B, depth=2) as p:
        assert p.push(xb[:4 * B], yb[:4 * B]) == b""           # push 0 in flight
        assert p.push(xb[4 * B:], yb[4 * B:]) == want[:len(want) // 2]   # push 0s 4 blocks
        assert p.flush() == want[len(want) // 2:]
    L = _lib.lib()
    h = L.bx_pipe_create_async(q, n, 4 * B, 0, 2)
    try:
        got = ctypes.c_int64()
        one = (ctypes.c_uint8 * 1)()
        assert L.bx_pipe_push(h, xb, yb, 4 * B, None, 0, ctypes.byref(got)) == 0
        assert L.bx_pipe_flush(h, one, ctypes.byref(got)) == _lib.BX_EINVAL
        assert b"drain first" in L.bx_last_error()
        assert L.bx_pipe_push(h, xb, yb, 4 * B, one, 1, ctypes.byref(got)) == _lib.BX_EINVAL
        assert b"out_cap" in L.bx_last_error()
        assert L.bx_pipe_push(h, xb, yb, 5 * B, one, 1, ctypes.byref(got)) == _lib.BX_EINVAL
        assert b"chunk_bytes" in L.bx_last_error()
    finally:
        L.bx_pipe_destroy(h)


def test_custom_modulus_contexts():
    """GFContext with a non-default irreducible modulus multiplies on the GPU."""
    from oracle import pyoracle
    rnd = random.Random(41)

    def other_modulus(q):
        # an irreducible modulus different from the shipped one (scan from the top)
        default = bx.modulus_int(q)
        for k in range(q - 1, 0, -1):
            m = (1 << q) | (1 << k) | 1
            if m != default and bx.is_irreducible(m):
                return m
        for a_ in range(q - 1, 3, -1):
            for b_ in range(a_ - 1, 1, -1):
                m = (1 << q) | (1 << a_) | (1 << b_) | 0b11
                if m != default and bx.is_irreducible(m):
                    return m
        return None

    for q in (3, 8, 13, 64, 100, 127):
        mod = other_modulus(q)
        assert mod is not None
        ctx = bx.GFContext(q, modulus=mod)
        a = [rnd.getrandbits(q) for _ in range(20)]
        b = [rnd.getrandbits(q) for _ in range(20)]
        want = [pyoracle.gf_mul(q, mod, x, y) for x, y in zip(a, b)]
        assert ctx.mul_many(a, b) == want, q
        assert ctx.mul(a[0], b[0]) == want[0]
        xs, ys = a[:7], b[:7]
        ip = 0
        for x, y in zip(xs, ys):
            ip ^= pyoracle.gf_mul(q, mod, x, y)
        assert bx.ext_ip(ctx, xs, ys) == ip
