"""Host-side logic on CPU: plans, reports, BitReader replay, sharding ranges,
and that libbx_b200.so loads and exports every symbol of include/blockext_b200.h.

The device compute is replaced, in this module only, by the CPU oracle through
monkeypatching sharding.extract_packed -- so the bookkeeping (consumed bits,
discarded tails, stop reasons, cursor, pad bits) is checked against the
reference's recorded reports without a GPU.
"""
import io
import re
from fractions import Fraction

import pytest

import paper_2402_14607_b200 as bx
from paper_2402_14607_b200 import _lib, sharding
from oracle import coracle

from bxtest_util import DribbleIO, case_inputs, place, report_dict, tiny_eq_plan
from conftest import REPO


@pytest.fixture
def oracle_compute(monkeypatch):
    def fake(xv, yv, q, n, count, *, x_bit0=0, y_bit0=0, device=None, devices=None, out=None):
        xb = bytes(memoryview(xv).cast("B")) if not hasattr(xv, "numpy") else xv.numpy().tobytes()
        yb = bytes(memoryview(yv).cast("B")) if not hasattr(yv, "numpy") else yv.numpy().tobytes()
        return place(coracle.extract_eq(xb, yb, q, n, count, x_bit0=x_bit0, y_bit0=y_bit0), out)
    monkeypatch.setattr(sharding, "extract_packed", fake)

    def fake_neq(xv, yv, q1, step, n, count, *, device=None):
        xb = bytes(memoryview(xv).cast("B")) if not hasattr(xv, "numpy") else xv.numpy().tobytes()
        yb = bytes(memoryview(yv).cast("B")) if not hasattr(yv, "numpy") else yv.numpy().tobytes()
        acc, pos, off = 0, 0, 0
        for k in range(count):
            q = q1 + k * step
            z = coracle.extract_eq(xb, yb, q, n, 1, x_bit0=off, y_bit0=off)
            acc |= int.from_bytes(z, "little") << pos
            pos += q
            off += q * n
        return acc.to_bytes((pos + 7) // 8, "little")
    monkeypatch.setattr(sharding, "extract_neq_packed", fake_neq)


def test_header_symbols_exported():
    hdr = (REPO / "include" / "blockext_b200.h").read_text()
    declared = set(re.findall(r"^\w[\w\s\*]*?\b(bx_\w+)\(", hdr, re.M))
    assert declared == set(_lib.SIGNATURES), declared ^ set(_lib.SIGNATURES)
    L = _lib.lib()
    for name in declared:
        assert hasattr(L, name)
    assert L.bx_version() == 100


def test_abi_modulus_table_matches_reference(golden):
    ref = golden("moduli.json")
    for q in range(1, 129):
        assert list(_lib.modulus_exponents(q)) == ref[str(q)]
    with pytest.raises(bx.CapacityError):
        _lib.modulus_exponents(129)


def test_abi_argument_errors_without_gpu():
    L = _lib.lib()
    assert L.bx_extract_eq(None, 0, 0, None, 0, 0, 129, 4, 1, None, 0, None) == _lib.BX_ERANGE
    assert L.bx_extract_eq(None, 0, 0, None, 0, 0, 4, 0, 1, None, 0, None) == _lib.BX_EINVAL
    assert L.bx_extract_eq(None, 0, 0, None, 0, 0, 4, 4, 0, None, 0, None) == _lib.BX_OK
    assert L.bx_pack(None, 3, 8, 1, None, 0, None) == _lib.BX_EINVAL
    with pytest.raises(ValueError, match="shorter"):
        _lib.check(L.bx_extract_eq(1024, 4, 0, 1024, 4, 0, 4, 64, 1, 1024, 0, None), "x")


def test_launch_info_geometry():
    for q in (1, 4, 8, 9, 16, 32, 56, 58, 80, 128):
        for n in (1, 4, 64, 120, 2000):
            li = _lib.launch_info(q, n, 10_000)
            assert li["threads"] == li["tpb"] * li["tile"]
            assert li["threads"] % 32 == 0 and li["threads"] <= 256
            assert li["family"] == ("diag" if q <= 8 else "holes")
            # one-thread-per-block kernels: eq_direct_kernel (powers of two) and
            # eq_period_kernel (q = 24, 40, 48, 56), for 128-bit-aligned blocks
            assert li["direct"] == (q in (1, 2, 4, 8, 16, 32, 64, 128, 24, 40, 48, 56)
                                    and q * n % 128 == 0)
            ntiles = -(-10_000 // li["tile"])
            # small direct blocks (q <= 4, one or two 128-bit units) take two
            # blocks per thread (bx_core.cuh direct_bpt)
            bpt = 2 if li["direct"] and q <= 4 and q * n // 128 in (1, 2) else 1
            if li["tma"]:
                assert 0 < li["grid"] <= ntiles and li["staged"]
            else:
                assert li["grid"] == -(-ntiles // bpt)


def test_golden_plans_and_bounds(golden):
    for c in golden("eq_cases.json"):
        plan = tiny_eq_plan(bx, c["b"], c["samples"], c.get("rate", "3/4"), c["n"], c["q"])
        assert repr(plan.log2_error) == c["plan_log2_error"]


def test_plan_eq_reference_values():
    p = bx.plan_eq(16, 2**47, Fraction(1074, 1600), Fraction(1, 2**30))
    assert (p.vec_len, p.field_bits, p.num_blocks) == (71, 80, 2**51 // (80 * 71))
    p = bx.plan_eq(8, 2**28, "3/4", "2^-30")
    assert (p.vec_len, p.field_bits, p.num_blocks) == (48, 56, 798915)
    with pytest.raises(bx.UnsupportedRateError):
        bx.plan_eq(8, 100, "1/2", "2^-10")
    with pytest.raises(TypeError):
        bx.plan_eq(8, 100, 0.75, "2^-10")
    with pytest.raises(bx.DivergenceError):
        bx.error_bound_neq(bx.plan_neq(8, "3/4", 8, 0))


def test_report_text_round_trip():
    plan = tiny_eq_plan(bx, 8, 300, "3/4", 5, 8)
    rep = bx.ExtractionReport("eq", plan, 3, 120, 120, 24, 0, 0, -1.5, 0.25, True, "completed", 0)
    assert bx.ExtractionReport.from_text(rep.to_text()) == rep
    nplan = bx.plan_neq(8, "3/4", 8, 1)
    assert bx.plan_from_text(bx.plan_to_text(nplan)) == nplan


@pytest.mark.parametrize("which", ["eq"])
def test_eq_reports_match_reference(golden, oracle_compute, which):
    for c in golden("eq_cases.json"):
        xb, yb = case_inputs(c)
        plan = tiny_eq_plan(bx, c["b"], c["samples"], c.get("rate", "3/4"), c["n"], c["q"])
        sink = io.BytesIO()
        rep = bx.extract_eq(xb, yb, plan, max_blocks=c.get("max_blocks")).run(sink)
        assert sink.getvalue().hex() == c["out"], c["tag"]
        assert report_dict(rep) == c["report"], c["tag"]


def test_eq_reports_file_streams(golden, oracle_compute):
    # file-like inputs (BytesIO and 7-byte dribbles) replay the same reads
    for c in golden("eq_cases.json")[-12:]:
        xb, yb = case_inputs(c)
        plan = tiny_eq_plan(bx, c["b"], c["samples"], c.get("rate", "3/4"), c["n"], c["q"])
        for mk in (io.BytesIO, lambda d: DribbleIO(d, 7)):
            sink = io.BytesIO()
            rep = bx.extract_eq(mk(xb), mk(yb), plan, max_blocks=c.get("max_blocks")).run(sink)
            assert sink.getvalue().hex() == c["out"], c["tag"]
            if mk is io.BytesIO:
                assert report_dict(rep) == c["report"], c["tag"]


def test_eq_reports_mapped_files(golden, oracle_compute, tmp_path, monkeypatch):
    """Regular files are memory-mapped and replayed in closed form: same bytes
    and report as the reference, and each file is left at the position the
    reference's read() calls would have left it (as a BytesIO source shows)."""
    from paper_2402_14607_b200 import extractor as E
    monkeypatch.setattr(E._Source, "MAP_MIN_BYTES", 0)
    for c in golden("eq_cases.json")[-12:]:
        xb, yb = case_inputs(c)
        if not xb or not yb:
            continue
        plan = tiny_eq_plan(bx, c["b"], c["samples"], c.get("rate", "3/4"), c["n"], c["q"])
        bx_, by_ = io.BytesIO(xb), io.BytesIO(yb)
        bx.extract_eq(bx_, by_, plan, max_blocks=c.get("max_blocks")).run(io.BytesIO())
        (tmp_path / "x").write_bytes(b"HDR" + xb)
        (tmp_path / "y").write_bytes(yb)
        with open(tmp_path / "x", "rb") as fx, open(tmp_path / "y", "rb") as fy:
            fx.read(3)                               # start mid-file
            run = bx.extract_eq(fx, fy, plan, max_blocks=c.get("max_blocks"))
            assert run._x._pos_file is fx           # the mapped path is the one under test
            sink = io.BytesIO()
            rep = run.run(sink)
            assert sink.getvalue().hex() == c["out"], c["tag"]
            assert report_dict(rep) == c["report"], c["tag"]
            assert (fx.tell() - 3, fy.tell()) == (bx_.tell(), by_.tell()), c["tag"]
    # one file object feeding both streams: read alternately, never mapped
    c = golden("eq_cases.json")[-1]
    xb, yb = case_inputs(c)
    plan = tiny_eq_plan(bx, c["b"], c["samples"], c.get("rate", "3/4"), c["n"], c["q"])
    both = io.BytesIO(xb + yb)
    want = bx.extract_eq(both, both, plan).run(io.BytesIO())
    (tmp_path / "xy").write_bytes(xb + yb)
    with open(tmp_path / "xy", "rb") as f:
        run = bx.extract_eq(f, f, plan)
        assert run._x._mem is None
        assert report_dict(run.run(io.BytesIO())) == report_dict(want)
        assert f.tell() == both.tell()


def test_neq_reports_match_reference(golden, oracle_compute):
    for c in golden("neq_cases.json"):
        if c.get("zeros"):
            xb = yb = bytes(c["x_len"])
        else:
            xb, yb = case_inputs(c)
        plan = bx.plan_neq(c["b"], "3/4", c["q1"], c["growth"])
        sink = io.BytesIO()
        rep = bx.extract_neq(xb, yb, plan, max_blocks=c["max_blocks"]).run(sink)
        assert sink.getvalue().hex() == c["out"], c
        assert report_dict(rep) == c["report"], c


def test_iteration_chunks_and_segments(golden, oracle_compute):
    c = next(c for c in golden("eq_cases.json") if c["tag"] == "multi_fill")
    xb, yb = case_inputs(c)
    plan = tiny_eq_plan(bx, c["b"], c["samples"], "3/4", c["n"], c["q"])
    run = bx.extract_eq(xb, yb, plan, segment_blocks=640)
    chunks = list(run)
    assert [ch.index for ch in chunks[:3]] == [1, 2, 3]
    acc = 0
    for k, ch in enumerate(chunks):
        assert ch.width == c["q"]
        acc |= ch.bits << (k * c["q"])
    assert acc.to_bytes(len(c["out"]) // 2, "little").hex() == c["out"]
    assert run.report.blocks_completed == len(chunks)
    assert run.cursor.block_index == len(chunks) + 1
    with pytest.raises(RuntimeError):
        list(run)


@pytest.mark.parametrize("kind", ["bytes", "file", "dribble"])
def test_multi_segment_run_single_buffer(golden, oracle_compute, tmp_path, kind):
    """run(sink) over several segments: whole-run output buffer (in-memory and
    regular-file sources, size known) or per-segment parts (pipe-like source):
    the same bytes, one sink write, same report."""
    c = next(c for c in golden("eq_cases.json") if c["tag"] == "multi_fill")
    xb, yb = case_inputs(c)
    plan = tiny_eq_plan(bx, c["b"], c["samples"], "3/4", c["n"], c["q"])
    want = bx.extract_eq(xb, yb, plan).run(io.BytesIO())
    if kind == "bytes":
        src = (xb, yb)
    elif kind == "file":
        (tmp_path / "x").write_bytes(xb)
        (tmp_path / "y").write_bytes(yb)
        src = (open(tmp_path / "x", "rb"), open(tmp_path / "y", "rb"))
    else:
        src = (DribbleIO(xb, 1000), DribbleIO(yb, 777))

    class OneWrite(io.BytesIO):
        writes = 0

        def write(self, b):
            OneWrite.writes += 1
            return super().write(b)

    sink = OneWrite()
    run = bx.extract_eq(*src, plan, segment_blocks=640)
    rep = run.run(sink)
    if kind == "file":
        for f in src:
            f.close()
    assert sink.getvalue().hex() == c["out"]
    assert OneWrite.writes == 1
    assert report_dict(rep) == report_dict(want)


def test_type_checks():
    plan = tiny_eq_plan(bx, 8, 100, "3/4", 5, 8)
    nplan = bx.plan_neq(8, "3/4", 8, 1)
    with pytest.raises(TypeError):
        bx.extract_eq(b"", b"", nplan)
    with pytest.raises(TypeError):
        bx.extract_neq(b"", b"", plan)


def test_shard_ranges():
    for nb in (0, 1, 63, 64, 65, 1000, 8388608, 4194305):
        for parts in (1, 2, 3, 4, 8):
            rs = sharding.shard_ranges(nb, parts)
            assert len(rs) == parts
            assert sum(c for _, c in rs) == nb
            pos = 0
            for s, c in rs:
                if c:
                    assert s == pos and s % 64 == 0
                    pos += c


def test_gf_context_validation():
    with pytest.raises(bx.CapacityError):
        bx.GFContext(129)
    with pytest.raises(ValueError):
        bx.GFContext(2, modulus=0b101)
    with pytest.raises(ValueError):
        bx.GFContext(2, modulus=0b110)
    ctx = bx.field(4)
    with pytest.raises(ValueError):
        ctx.add(16, 0)
    assert ctx.add(5, 3) == 6
    assert bx.field(80) is bx.field(80)
    assert bx.is_irreducible(0b111) and not bx.is_irreducible(0b101)


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    plan = tiny_eq_plan(bx, 8, 100, "3/4", 5, 8)
    with pytest.raises(bx.DeviceError):
        bx.extract_eq(bytes(100), bytes(100), plan).run()
    with pytest.raises(bx.DeviceError):
        bx.ext_ip(bx.field(4), (1,), (2,))


def test_bitio_reader_writer():
    from paper_2402_14607_b200.bitio import BitReader, BitWriter, unpack_values
    from bxtest_util import DribbleIO
    r = BitReader(bytes([0b10110010]))
    assert [r.read_bits(1) for _ in range(8)] == [0, 1, 0, 0, 1, 1, 0, 1]
    r = BitReader(bytes([0xAB, 0xCD]))
    assert r.read_bits(12) == 0xDAB and r.read_bits(4) == 0xC and r.read_bits(1) is None
    r = BitReader(bytes([0xFF]))
    assert r.read_bits(5) == 0b11111 and r.read_bits(5) is None
    assert r.tail_bits() == 3 and r.bits_consumed == 5
    data = bytes(range(40))
    a, b = BitReader(data), BitReader(DribbleIO(data, 3))
    while True:
        va, vb = a.read_bits(13), b.read_bits(13)
        assert va == vb
        if va is None:
            assert a.tail_bits() == b.tail_bits()
            break
    w = BitWriter()
    w.write_bits(0b101, 3)
    assert w.getvalue() == (bytes([0b101]), 5)
    with pytest.raises(ValueError):
        w.write_bits(4, 2)
    assert unpack_values(bytes([0x21, 0x43]), 4, 4) == [1, 2, 3, 4]
