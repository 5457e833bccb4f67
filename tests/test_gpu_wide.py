"""GF(2^256) extraction (config 3 as BASELINE states it: 1024-bit blocks,
m = 256) -- the opt-in extension beyond the reference's q <= 128 cap
(pkg/src/blockext/gf2q.py:111-112).

Parity: the width-agnostic restatement (oracle/pyoracle.py: poly_mul +
fold-table reduction, gf2q.py:44-54,124-133,156-169, pinned against the
reference for every q <= 128 in test_oracle.py) evaluated at q = 256 with the
modulus the reference's scan order picks; plus algebraic identities at full
size (bilinearity, symmetry, the unit element)."""
import random

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from paper_2402_14607_b200 import _lib
from paper_2402_14607_b200 import device as D
from paper_2402_14607_b200 import wide
from paper_2402_14607_b200 import workloads as W
from oracle import pyoracle

pytestmark = pytest.mark.gpu
Q = 256
MOD = wide.modulus_int(Q)


def _want(xb: bytes, yb: bytes, n: int, k: int) -> bytes:
    return pyoracle.extract_eq(xb, yb, Q, n, k, MOD)


@pytest.mark.parametrize("n,k", [(1, 1), (1, 257), (2, 130), (3, 65), (4, 200), (5, 31), (8, 40)])
def test_wide_random_vs_width_agnostic_oracle(n, k):
    rnd = random.Random(n * 1000 + k)
    nb = k * Q * n // 8
    xb, yb = rnd.randbytes(nb), rnd.randbytes(nb)
    assert wide.extract_eq_wide(xb, yb, n, k) == _want(xb, yb, n, k)


def test_wide_special_elements():
    """all-ones, zero, and the unit element (x_0 = 1: output = y_0 reduced)."""
    n = 4
    ones = bytes([0xFF]) * (Q * n // 8)
    zero = bytes(Q * n // 8)
    assert wide.extract_eq_wide(ones, ones, n, 1) == _want(ones, ones, n, 1)
    assert wide.extract_eq_wide(zero, ones, n, 1) == bytes(Q // 8)
    rnd = random.Random(3)
    y = rnd.randbytes(Q * n // 8)
    unit = (1).to_bytes(Q // 8, "little") + bytes((n - 1) * Q // 8)
    assert wide.extract_eq_wide(unit, y, n, 1) == y[:Q // 8]


def test_wide_device_inputs_and_errors():
    rnd = random.Random(9)
    n, k = 4, 300
    xb, yb = rnd.randbytes(k * 128), rnd.randbytes(k * 128)
    xd, _ = D.to_device_stream(xb, "cuda")
    yd, _ = D.to_device_stream(yb, "cuda")
    assert wide.extract_eq_wide(xd[:k * 128], yd[:k * 128], n) == wide.extract_eq_wide(xb, yb, n)
    with pytest.raises(Exception):
        wide.extract_eq_wide(xb, yb, n, k + 1)        # more blocks than the inputs hold
    L = _lib.lib()
    assert L.bx_extract_eq_wide(xd.data_ptr(), 512, yd.data_ptr(), 512, 128, 4, 1,
                                xd.data_ptr(), 0, None) == _lib.BX_ERANGE


def test_c3_as_stated_full_size():
    """Config 3 at its stated size and shape: 2 x 2^32 Bernoulli(0.3) bits
    (seeds 1, 2), 1024-bit blocks, q = 256, n = 4 -> 4,194,304 blocks.
    Sampled blocks (edges + random) vs the oracle on the same windows, and
    bilinearity over the whole run: E(x, y) ^ E(x, y') == E(x, y ^ y')."""
    wl = W.WORKLOADS["c3"]
    n = 4
    xd, nbytes = W.stream_device(wl.x, wl.samples, "cuda")
    yd, _ = W.stream_device(wl.y, wl.samples, "cuda")
    k = nbytes * 8 // (Q * n)
    assert k == 2**32 // 1024
    out = wide.extract_eq_wide(xd[:nbytes], yd[:nbytes], n)
    assert len(out) == k * Q // 8
    xh = xd[:nbytes].cpu().numpy()
    yh = yd[:nbytes].cpu().numpy()
    rnd = np.random.default_rng(5)
    for l in [0, 1, k // 2, k - 2, k - 1] + rnd.integers(0, k, 20).tolist():
        lo, hi = l * 128, (l + 1) * 128
        got = out[l * 32:(l + 1) * 32]
        assert got == _want(xh[lo:hi].tobytes(), yh[lo:hi].tobytes(), n, 1), l
    y2 = torch.randint(0, 256, (nbytes,), dtype=torch.uint8, device="cuda")
    e2 = wide.extract_eq_wide(xd[:nbytes], y2, n)
    e12 = wide.extract_eq_wide(xd[:nbytes], yd[:nbytes] ^ y2, n)
    a = np.frombuffer(out, np.uint8) ^ np.frombuffer(e2, np.uint8)
    assert np.array_equal(a, np.frombuffer(e12, np.uint8))
