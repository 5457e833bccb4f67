"""The raw-sample packer (reference sources._pack_samples, pkg/src/blockext/
sources.py:116-121) through bx_pack, for every (sample type, width) the tile
kernel is instantiated for, against the C oracle (bxo_pack).

Covers: whole and partial 1024-sample warp tiles, a single sample, word- and
non-word-aligned destinations (the funnel-shifted store and the atomic merge of
shared boundary words), bits outside the range preserved (canary), the
full-width copy path, unaligned sample pointers (generic kernel) and the
narrowing of over-wide sample types in device.pack.
"""
import random

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from paper_2402_14607_b200 import _lib
from paper_2402_14607_b200 import device as D
from oracle import coracle

pytestmark = pytest.mark.gpu

NATURAL = ([(1, b) for b in range(1, 9)] + [(2, b) for b in range(1, 17)]
           + [(4, b) for b in range(17, 33)] + [(8, b) for b in range(33, 65)])
COUNTS = (1, 1023, 1024, 1025, 5 * 1024 + 17)
OFFSETS = (0, 5, 32, 37)
CANARY = 0xA5


def _oracle_int(vals: np.ndarray, b: int) -> int:
    want = coracle.pack([int(v) & ((1 << b) - 1) for v in vals.tolist()], b)
    return int.from_bytes(want, "little")


def _check(t: torch.Tensor, vals: np.ndarray, b: int, off: int, what):
    cnt = vals.size
    end = off + cnt * b
    nbytes = D.padded_len((end + 7) // 8 + 8)
    buf = torch.full((nbytes,), CANARY, dtype=torch.uint8, device="cuda")
    D.pack(t, b, out=buf, out_bit0=off)
    got = int.from_bytes(buf.cpu().numpy().tobytes(), "little")
    rng_mask = ((1 << (cnt * b)) - 1) << off
    assert (got & rng_mask) >> off == _oracle_int(vals, b), what
    canary = int.from_bytes(bytes([CANARY]) * nbytes, "little")
    assert got & ~rng_mask == canary & ~rng_mask, ("canary", what)


@pytest.mark.parametrize("elem,b", NATURAL)
def test_pack_tile_kernel_vs_oracle(elem, b):
    rnd = np.random.default_rng(elem * 100 + b)
    dt = np.dtype(f"u{elem}")
    for cnt in COUNTS:
        vals = rnd.integers(0, np.iinfo(dt).max, size=cnt, dtype=dt, endpoint=True)
        t = torch.from_numpy(vals.view(np.dtype(f"i{elem}"))).cuda()
        for off in OFFSETS:
            _check(t, vals, b, off, (elem, b, cnt, off))


def test_pack_full_width_is_a_copy_and_launches_no_kernel():
    rnd = np.random.default_rng(3)
    for elem in (1, 2, 4, 8):
        dt = np.dtype(f"u{elem}")
        vals = rnd.integers(0, np.iinfo(dt).max, size=4097, dtype=dt, endpoint=True)
        t = torch.from_numpy(vals.view(np.dtype(f"i{elem}"))).cuda()
        n0 = _lib.launch_count()
        _check(t, vals, 8 * elem, 16, elem)
        assert _lib.launch_count() == n0, "full-width byte-aligned pack launched a kernel"
        _check(t, vals, 8 * elem, 3, elem)   # not byte aligned: a kernel


def test_pack_unaligned_samples_and_wide_types():
    """Sample pointers off the 32-byte grid and sample types wider than b
    needs (uint64 samples of 6 bits, int16 Markov states of 1 bit)."""
    rnd = np.random.default_rng(4)
    vals = rnd.integers(0, 255, size=9000, dtype=np.uint8, endpoint=True)
    base = torch.from_numpy(vals).cuda()
    for lead in (1, 3, 17):
        _check(base[lead:], vals[lead:], 6, 11, ("unaligned", lead))
    for elem, b in ((8, 6), (8, 14), (4, 3), (2, 1), (4, 12), (8, 31)):
        dt = np.dtype(f"u{elem}")
        v = rnd.integers(0, np.iinfo(dt).max, size=7000, dtype=dt, endpoint=True)
        t = torch.from_numpy(v.view(np.dtype(f"i{elem}"))).cuda()
        _check(t, v, b, 0, ("wide", elem, b))
        _check(t, v, b, 9, ("wide", elem, b))


def test_pack_large_random_chunks_round_trip():
    """A 2^24-sample chunk (generate()'s DRAW_CHUNK) at each bench width,
    unpacked again on the host with numpy."""
    rnd = np.random.default_rng(5)
    for elem, b in ((1, 1), (1, 6), (2, 12), (2, 14)):
        dt = np.dtype(f"u{elem}")
        vals = rnd.integers(0, (1 << b) - 1, size=1 << 24, dtype=dt, endpoint=True)
        t = torch.from_numpy(vals.view(np.dtype(f"i{elem}"))).cuda()
        out = D.pack(t, b)
        nbytes = ((1 << 24) * b + 7) // 8
        bits = np.unpackbits(out[:nbytes].cpu().numpy(), bitorder="little")
        back = bits.reshape(-1, b).astype(np.uint64) @ (1 << np.arange(b, dtype=np.uint64))
        assert np.array_equal(back, vals.astype(np.uint64)), (elem, b)
