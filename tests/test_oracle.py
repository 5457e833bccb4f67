"""The CPU oracle against the reference's own outputs (tests/golden/*).

These pin the oracle before it is trusted as the checker for the GPU kernels.
"""
import hashlib
import random

import numpy as np
import pytest

from oracle import coracle, pyoracle


@pytest.fixture(scope="module")
def moduli(golden):
    return {int(k): v for k, v in golden("moduli.json").items()}


def test_generated_moduli_match_reference(moduli):
    from paper_2402_14607_b200._moduli_data import MIDDLE_EXPONENTS
    rows = MIDDLE_EXPONENTS.split(";")
    assert len(rows) == 128
    for q in range(1, 129):
        mids = [int(t) for t in rows[q - 1].split(",") if t]
        assert [q] + mids + [0] == moduli[q], q


def test_header_table_matches_reference(moduli):
    import re
    from conftest import REPO
    text = (REPO / "paper_2402_14607_b200/csrc/bx_moduli.h").read_text()
    rows = re.findall(r"\{(\d), \{([\d, ]+)\}\},\s+// q=(\d+)", text)
    assert len(rows) == 128
    for cnt, exps, q in rows:
        e = [int(t) for t in exps.split(",")][: int(cnt)]
        assert e == moduli[int(q)]


def test_gf_mul_kats(golden, moduli):
    kats = golden("gf_mul.json")
    for q in range(1, 129):
        rows = kats[str(q)]
        a = [int(r[0], 16) for r in rows]
        b = [int(r[1], 16) for r in rows]
        want = [int(r[2], 16) for r in rows]
        assert coracle.gf_mul(q, a, b) == want, q
        m = pyoracle.modulus_int(moduli[q])
        assert [pyoracle.gf_mul(q, m, x, y) for x, y in zip(a, b)] == want, q


def test_ext_ip_kats(golden, moduli):
    for c in golden("ext_ip.json"):
        q = c["q"]
        xs = [int(v, 16) for v in c["x"]]
        ys = [int(v, 16) for v in c["y"]]
        assert pyoracle.ext_ip(q, pyoracle.modulus_int(moduli[q]), xs, ys) == int(c["z"], 16)


def _case_inputs(c):
    rng = np.random.default_rng(c["seed"])
    return rng.bytes(c["x_len"]), rng.bytes(c["y_len"])


@pytest.mark.parametrize("mode", [0, 1])
def test_eq_cases(golden, mode):
    for c in golden("eq_cases.json"):
        xb, yb = _case_inputs(c)
        k = c["report"]["blocks_completed"]
        if k == 0:
            assert c["out"] == ""
            continue
        got = coracle.extract_eq(xb, yb, c["q"], c["n"], k, mode=mode)
        assert got.hex() == c["out"], c["tag"]


def test_eq_cases_pyoracle_small(golden, moduli):
    for c in golden("eq_cases.json")[:128:9]:
        xb, yb = _case_inputs(c)
        k = c["report"]["blocks_completed"]
        m = pyoracle.modulus_int(moduli[c["q"]])
        assert pyoracle.extract_eq(xb, yb, c["q"], c["n"], k, m).hex() == c["out"]


def test_pack_kats(golden):
    for c in golden("pack.json"):
        vals = [int(v, 16) for v in c["values"]]
        assert coracle.pack(vals, c["b"]).hex() == c["out"]
        assert pyoracle.pack(vals, c["b"]).hex() == c["out"]


def test_c1_full(golden):
    from paper_2402_14607_b200 import workloads as W
    meta = golden("c1.json")
    wl = W.WORKLOADS["c1"]
    xb = W.stream_bytes_host(wl.x, wl.samples).tobytes()
    yb = W.stream_bytes_host(wl.y, wl.samples).tobytes()
    assert hashlib.sha256(xb).hexdigest() == meta["x_sha256"]
    assert hashlib.sha256(yb).hexdigest() == meta["y_sha256"]
    out = coracle.extract_eq(xb, yb, wl.q, wl.n, wl.num_blocks)
    assert out == golden("c1_out.bin")
    assert coracle.extract_eq(xb, yb, wl.q, wl.n, wl.num_blocks, mode=0) == out


def test_sampled_blocks(golden):
    from paper_2402_14607_b200 import workloads as W
    for name, rec in golden("sampled.json").items():
        wl = W.WORKLOADS[name]
        B = wl.block_bits
        for l, z in rec["blocks"][:4]:
            b = wl.b
            s0 = (l * B) // b
            s1 = -(-((l + 1) * B) // b)
            if b == 1:
                s0 -= s0 % 8
                s1 += (-s1) % 8
            xw = W.window_bytes(wl.x, s0 * b, (s1 - s0) * b)
            yw = W.window_bytes(wl.y, s0 * b, (s1 - s0) * b)
            skip = l * B - s0 * b
            got = coracle.extract_eq(xw, yw, wl.q, wl.n, 1, x_bit0=skip, y_bit0=skip)
            assert int.from_bytes(got, "little") == int(z, 16), (name, l)


def test_modes_agree_random_shapes():
    rnd = random.Random(5)
    for _ in range(60):
        q = rnd.randint(1, 128)
        n = rnd.randint(1, 20)
        k = rnd.randint(1, 30)
        nb = (k * q * n + 7) // 8 + 3
        xb, yb = rnd.randbytes(nb), rnd.randbytes(nb)
        off = rnd.randint(0, 13)
        a = coracle.extract_eq(xb, yb, q, n, k, x_bit0=off, y_bit0=off, mode=0)
        b = coracle.extract_eq(xb, yb, q, n, k, x_bit0=off, y_bit0=off, mode=1)
        assert a == b
