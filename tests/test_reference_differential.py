"""Randomised differential tests against the LIVE reference (CPU only).

Runs only where the reference package is importable (the build container,
/root/reference); skipped elsewhere.  The device compute is replaced by the
CPU oracle (test-only monkeypatch), so what is compared is the drop-in's host
behaviour -- BitReader replay, stop reasons, discarded-bit accounting, cursor,
reports, output framing -- on random plans, stream lengths and read patterns.
"""
import io
import pathlib
import random
import sys

import pytest
from hypothesis import given, settings, strategies as st

REF = pathlib.Path("/root/reference/pkg/src")
if not REF.exists():
    pytest.skip("reference not available", allow_module_level=True)
sys.path.insert(0, str(REF))

import blockext as R  # noqa: E402

import paper_2402_14607_b200 as bx  # noqa: E402
from paper_2402_14607_b200 import sharding  # noqa: E402
from oracle import coracle  # noqa: E402

from bxtest_util import DribbleIO, place, report_dict  # noqa: E402


@pytest.fixture(autouse=True)
def oracle_compute(monkeypatch):
    def fake(xv, yv, q, n, count, *, x_bit0=0, y_bit0=0, device=None, devices=None, out=None):
        return place(coracle.extract_eq(bytes(xv), bytes(yv), q, n, count, x_bit0=x_bit0,
                                        y_bit0=y_bit0), out)

    def fake_neq(xv, yv, q1, step, n, count, *, device=None):
        xb, yb = bytes(xv), bytes(yv)
        acc, pos, off = 0, 0, 0
        for k in range(count):
            q = q1 + k * step
            acc |= int.from_bytes(coracle.extract_eq(xb, yb, q, n, 1, x_bit0=off, y_bit0=off),
                                  "little") << pos
            pos += q
            off += q * n
        return acc.to_bytes((pos + 7) // 8, "little")
    monkeypatch.setattr(sharding, "extract_packed", fake)
    monkeypatch.setattr(sharding, "extract_neq_packed", fake_neq)


def _rep(r):
    d = report_dict(r)
    d["cursor"] = None
    return d


@settings(max_examples=60, deadline=None)
@given(st.data())
def test_eq_random_against_reference(data):
    b = data.draw(st.sampled_from([1, 2, 4, 8, 16]))
    q = data.draw(st.integers(1, 128))
    n = data.draw(st.integers(1, 12))
    samples = data.draw(st.integers(1, 5000))
    xl = data.draw(st.integers(0, (samples * b + 7) // 8 + 70))
    yl = data.draw(st.integers(0, (samples * b + 7) // 8 + 70))
    maxb = data.draw(st.sampled_from([None, 1, 3, 17]))
    step = data.draw(st.sampled_from([None, 1, 5, 4096]))
    seed = data.draw(st.integers(0, 2**32))
    rnd = random.Random(seed)
    xb, yb = rnd.randbytes(xl), rnd.randbytes(yl)
    ref_plan = R.EqPlan(b, samples, R.params.as_rational("3/4"), R.params.as_rational("1/2"), n, q,
                        samples * b // (q * n), samples * b // (q * n) * q, 0.0)
    mk = (lambda d: d) if step is None else (lambda d: DribbleIO(d, step))
    s1, s2 = io.BytesIO(), io.BytesIO()
    r1 = R.extract_eq(mk(xb), mk(yb), ref_plan, max_blocks=maxb)
    rep1 = r1.run(s1)
    r2 = bx.extract_eq(mk(xb), mk(yb), ref_plan, max_blocks=maxb)   # the reference's own plan object
    rep2 = r2.run(s2)
    assert s1.getvalue() == s2.getvalue()
    assert report_dict(rep1) == report_dict(rep2)
    assert (r1.cursor.block_index, r1.cursor.sample_index, r1.cursor.field_bits) == \
        (r2.cursor.block_index, r2.cursor.sample_index, r2.cursor.field_bits)


@settings(max_examples=40, deadline=None)
@given(st.data())
def test_neq_random_against_reference(data):
    b = data.draw(st.sampled_from([1, 2, 4, 8]))
    growth = data.draw(st.integers(0, 3))
    q1 = b * data.draw(st.integers(1, max(1, 24 // b)))
    nbytes = data.draw(st.integers(0, 6000))
    maxb = data.draw(st.sampled_from([None, 1, 4, 9]))
    seed = data.draw(st.integers(0, 2**32))
    rnd = random.Random(seed)
    xb, yb = rnd.randbytes(nbytes), rnd.randbytes(max(0, nbytes - rnd.randint(0, 20)))
    rp = R.plan_neq(b, "3/4", q1, growth)
    s1, s2 = io.BytesIO(), io.BytesIO()
    r1 = R.extract_neq(xb, yb, rp, max_blocks=maxb)
    rep1 = r1.run(s1)
    r2 = bx.extract_neq(xb, yb, rp, max_blocks=maxb)
    rep2 = r2.run(s2)
    assert s1.getvalue() == s2.getvalue()
    assert report_dict(rep1) == report_dict(rep2)
    assert (r1.cursor.block_index, r1.cursor.sample_index, r1.cursor.field_bits) == \
        (r2.cursor.block_index, r2.cursor.sample_index, r2.cursor.field_bits)


@settings(max_examples=40, deadline=None)
@given(st.data())
def test_plans_and_bounds_against_reference(data):
    b = data.draw(st.sampled_from([1, 2, 4, 8, 16, 32]))
    num = data.draw(st.integers(51, 100))
    rate = f"{num}/100"
    n = data.draw(st.integers(1, 2**40))
    eps = f"2^-{data.draw(st.integers(1, 60))}"
    try:
        p1 = R.plan_eq(b, n, rate, eps)
    except Exception as exc:  # noqa: BLE001
        with pytest.raises(type(exc)):
            bx.plan_eq(b, n, rate, eps)
        return
    p2 = bx.plan_eq(b, n, rate, eps)
    assert p1.__dict__ == p2.__dict__
    assert R.plan_to_text(p1) == bx.plan_to_text(p2)
    g = data.draw(st.integers(0, 3))
    q1 = b * data.draw(st.integers(1, max(1, 128 // b)))
    n1 = R.plan_neq(b, rate, q1, g)
    n2 = bx.plan_neq(b, rate, q1, g)
    assert n1.__dict__ == n2.__dict__
    k = data.draw(st.integers(1, 40))
    assert R.error_bound_neq(n1, k) == bx.error_bound_neq(n2, k)


class _Recorder(io.BytesIO):
    """BytesIO that records every read(size) call."""

    def __init__(self, data):
        super().__init__(data)
        self.sizes = []

    def read(self, size=-1):
        self.sizes.append(size)
        return super().read(size)


@settings(max_examples=80, deadline=None)
@given(st.data())
def test_bitio_against_reference(data):
    """BitReader / BitWriter / unpack_values (reference bitio.py:16-108): same
    values, same read(size) sequence, same counters and tails."""
    from paper_2402_14607_b200 import bitio as B
    from blockext import bitio as RB

    raw = data.draw(st.binary(min_size=0, max_size=600))
    chunk = data.draw(st.sampled_from([1, 3, 16, 64, 1 << 16]))
    widths = data.draw(st.lists(st.integers(1, 200), min_size=1, max_size=40))
    a, b = _Recorder(raw), _Recorder(raw)
    ra, rb = B.BitReader(a, chunk), RB.BitReader(b, chunk)
    for w in widths:
        assert ra.read_bits(w) == rb.read_bits(w)
        assert (ra.bits_consumed, ra.tail_bits()) == (rb.bits_consumed, rb.tail_bits())
    assert a.sizes == b.sizes
    wa, wb = B.BitWriter(), RB.BitWriter()
    for w in widths:
        v = data.draw(st.integers(0, (1 << w) - 1))
        wa.write_bits(v, w)
        wb.write_bits(v, w)
        assert wa.bit_length == wb.bit_length
    assert wa.getvalue() == wb.getvalue()
    width = data.draw(st.integers(1, 128))
    count = data.draw(st.integers(0, 8 * len(raw) // width + 2))
    try:
        want = RB.unpack_values(raw, width, count)
    except ValueError:
        with pytest.raises(ValueError):
            B.unpack_values(raw, width, count)
    else:
        assert B.unpack_values(raw, width, count) == want
