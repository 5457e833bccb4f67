"""Verification suites: host helpers on CPU, the
exhaustive kernels on the GPU, both against the reference's recorded results
(tests/golden/verify.json)."""
import hashlib

import numpy as np
import pytest

import paper_2402_14607_b200 as bx
from paper_2402_14607_b200 import verify as V


def test_walsh_transform_matches_definition():
    rows = np.random.default_rng(0).integers(0, 50, size=(3, 8))
    got = V.walsh_transform(rows)
    for r in range(3):
        for a in range(8):
            assert got[r, a] == sum(int(rows[r, w]) * (-1) ** bin(a & w).count("1") for w in range(8))


def test_parity_table():
    assert all(V.parity_table(5)[v] == bin(v).count("1") % 2 for v in range(32))


def test_first_bit_rows_definition():
    from oracle import pyoracle
    for q in (1, 3, 5, 8):
        ctx = bx.field(q)
        brow = V.first_bit_rows(ctx)
        m = ctx.modulus
        for v in range(1 << q):
            for a in range(1 << q):
                fb = pyoracle.gf_mul(q, m, a, v) & 1
                assert fb == bin(a & int(brow[v])).count("1") % 2


def test_bijection_and_xor_lemma():
    for q in range(1, 9):
        assert V.check_first_bit_bijection(bx.field(q))
    with pytest.raises(bx.InfeasibleError):
        V.check_first_bit_bijection(bx.field(9))
    rng = np.random.default_rng(3)
    for q in (1, 2, 3, 4):
        j = rng.random((1 << q, 5))
        j /= j.sum()
        lhs, rhs = V.xor_lemma_sides(q, j)
        assert lhs <= rhs + 1e-12 and V.check_xor_lemma_instance(q, j)
    with pytest.raises(bx.InfeasibleError):
        V.xor_lemma_sides(5, np.ones((32, 1)) / 32)


def test_limits_raise():
    with pytest.raises(bx.InfeasibleError):
        V.check_hadamard(bx.field(9), 2)
    with pytest.raises(bx.InfeasibleError):
        V.ip_value_table(bx.field(13), 1)
    assert list(V.hadamard_instances(3)) == [(1, 1), (1, 2), (1, 3), (2, 1), (3, 1)]


gpu = pytest.mark.gpu


@pytest.fixture
def cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@gpu
def test_ip_tables_match_reference(golden, cuda):
    for key, digest in golden("verify.json")["tables"].items():
        q, n = map(int, key.split(","))
        z = V.ip_value_table(bx.field(q), n)
        assert hashlib.sha256(z.astype(np.uint16).tobytes()).hexdigest() == digest, key


@gpu
def test_bias_and_distance_match_reference(golden, cuda):
    g = golden("verify.json")
    for c in g["bias"]:
        r = V.check_one_bit_bias(bx.field(c["q"]), c["n"], c["k"], seed=c["seed"], sampled_pairs=60)
        assert repr(r.max_bias) == c["max_bias"] and repr(r.bound) == c["bound"]
        assert r.pairs_tested == c["pairs"] and r.exhaustive == c["exhaustive"] and r.holds
    rng = np.random.default_rng(77)
    for c in g["distance"]:
        size = 1 << (c["q"] * c["n"])
        px = rng.random(size) ** 4
        px /= px.sum()
        py = rng.random(size) ** 2
        py /= py.sum()
        r = V.check_extractor_distance(bx.field(c["q"]), c["n"], px, py)
        # float64 sums of 2^(2qn) weights in a different order (device scatter-add
        # vs numpy's sequential bincount); |out - 2^-q| cancels, so compare to 1e-9
        assert r.distance == pytest.approx(float(c["distance"]), rel=1e-9, abs=1e-15)
        assert repr(r.bound) == c["bound"] and repr(r.rate) == c["rate"]


@gpu
def test_hadamard_verdicts_match_reference(golden, cuda):
    for c in golden("verify.json")["hadamard"]:
        ctx = bx.field(c["q"])
        if c["direct"] is not None:
            assert V.check_hadamard(ctx, c["n"], method="direct") == c["direct"]
        assert V.check_hadamard(ctx, c["n"], method="counts") == c["counts"]


@gpu
def test_hadamard_full_sweep_16_bits(cuda):
    """The reference's slow acceptance sweep (pkg/tests/test_acceptance.py:107-112):
    every (q, n) with q*n <= 16 -- exhaustive on the GPU."""
    failures = [(q, n) for q, n in V.hadamard_instances(16) if not V.check_hadamard(bx.field(q), n)]
    assert failures == []


@gpu
def test_ip_table_against_ext_ip(cuda):
    from oracle import pyoracle
    for q, n in [(3, 2), (4, 3), (1, 7), (5, 2)]:
        ctx = bx.field(q)
        z = V.ip_value_table(ctx, n)
        mask = (1 << q) - 1
        rnd = np.random.default_rng(q)
        for x, y in rnd.integers(0, 1 << (q * n), size=(200, 2)):
            xs = [(int(x) >> (i * q)) & mask for i in range(n)]
            ys = [(int(y) >> (i * q)) & mask for i in range(n)]
            assert z[x, y] == pyoracle.ext_ip(q, ctx.modulus, xs, ys)
