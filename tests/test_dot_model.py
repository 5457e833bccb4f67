"""CPU model of the dot-product holes leaf (csrc/bx_core.cuh: dsplit_x, dsplit_y,
dot16x2, Dot::unreduced): the integer arithmetic of IDP.2A on holed operands,
restated in Python and compared with a plain carry-less product.

Pins the no-carry claim the kernels rest on: with 16-bit halves holed by
0x9249 / 0x2492 / 0x4924 and bytes holed by 0x49 / 0x92 / 0x24, every 3-bit
field of a two-term dot product holds a count <= 6, so its low bit is the
GF(2) coefficient.  Runs without a GPU."""
import random

MX = (0x92499249, 0x24922492, 0x49244924)      # two 16-bit halves per word
MY = (0x49494949, 0x92929292, 0x24242424)      # four bytes per word
FIELD = (0x49249249, 0x92492492, 0x24924924)   # low bit of every 3-bit field, class c


def clmul(a: int, b: int) -> int:
    r = 0
    while b:
        if b & 1:
            r ^= a
        a <<= 1
        b >>= 1
    return r


def dp2a(a: int, b: int, hi: bool) -> int:
    """dp2a.lo / dp2a.hi on unsigned operands with c = 0 (PTX ISA, dp2a)."""
    h0, h1 = a & 0xFFFF, a >> 16
    by = [(b >> (8 * i)) & 0xFF for i in range(4)]
    s = h0 * by[2] + h1 * by[3] if hi else h0 * by[0] + h1 * by[1]
    assert s < 1 << 32
    return s


def byte_perm(a: int, b: int, sel: int) -> int:
    src = [(a >> (8 * i)) & 0xFF for i in range(4)] + [(b >> (8 * i)) & 0xFF for i in range(4)]
    return sum(src[(sel >> (4 * i)) & 7] << (8 * i) for i in range(4))


def leaf(pairs) -> int:
    """XOR over packed pairs (x word, y word) of the two 16x16 carry-less
    products each pair holds, the way Dot<16> accumulates and finishes."""
    lo, hi = [0, 0, 0], [0, 0, 0]
    for xw, yw in pairs:
        yp = byte_perm(yw, 0, 0x3120)
        for c in range(3):
            for r in range(3):
                s = (c + 3 - r) % 3
                for acc, h in ((lo, False), (hi, True)):
                    d = dp2a(xw & MX[r], yp & MY[s], h)
                    # every 3-bit field of class c holds a count <= 6
                    for p in range(c, 32, 3):
                        assert (d >> p) & 7 <= 6
                    assert d & ~(FIELD[c] * 7) & 0xFFFFFFFF == 0
                    acc[c] ^= d
    lo_v = (lo[0] & FIELD[0]) | (lo[1] & FIELD[1]) | (lo[2] & FIELD[2])
    hi_v = (hi[0] & FIELD[0]) | (hi[1] & FIELD[1]) | (hi[2] & FIELD[2])
    return lo_v ^ (hi_v << 8)


def want(pairs) -> int:
    r = 0
    for xw, yw in pairs:
        r ^= clmul(xw & 0xFFFF, yw & 0xFFFF) ^ clmul(xw >> 16, yw >> 16)
    return r


def test_leaf_worst_cases():
    for xw in (0xFFFFFFFF, 0x0000FFFF, 0xFFFF0000, 0x92499249, 0xAAAA5555):
        for yw in (0xFFFFFFFF, 0x00FF00FF, 0xFF00FF00, 0x49249249, 0x5555AAAA):
            assert leaf([(xw, yw)]) == want([(xw, yw)])
    assert leaf([(0xFFFFFFFF, 0xFFFFFFFF)] * 64) == want([(0xFFFFFFFF, 0xFFFFFFFF)] * 64)


def test_leaf_random_blocks():
    rnd = random.Random(2402)
    for _ in range(60):
        pairs = [(rnd.getrandbits(32), rnd.getrandbits(32)) for _ in range(rnd.randint(1, 40))]
        assert leaf(pairs) == want(pairs)


def test_packing_selectors_of_wider_elements():
    """pack_x / pack_y of Dot<Q>: halves of two elements side by side, and the
    matching byte order on the y side."""
    a, b = 0x44332211, 0x88776655
    assert byte_perm(a, b, 0x5410) == 0x66552211      # [b.lo16 : a.lo16]
    assert byte_perm(a, b, 0x7632) == 0x88774433      # [b.hi16 : a.hi16]
    assert byte_perm(a, b, 0x5140) == 0x66225511      # [b.b1, a.b1, b.b0, a.b0]
    assert byte_perm(a, b, 0x7362) == 0x88447733      # [b.b3, a.b3, b.b2, a.b2]
    # a 32-bit product through three Karatsuba leaves of packed halves
    rnd = random.Random(5)
    for _ in range(40):
        xa, xb, ya, yb = (rnd.getrandbits(32) for _ in range(4))
        xl, xh = byte_perm(xa, xb, 0x5410), byte_perm(xa, xb, 0x7632)
        yl, yh = byte_perm(ya, yb, 0x5140), byte_perm(ya, yb, 0x7362)

        def leaf_packed(xw, yp):
            lo, hi = [0, 0, 0], [0, 0, 0]
            for c in range(3):
                for r in range(3):
                    s = (c + 3 - r) % 3
                    lo[c] ^= dp2a(xw & MX[r], yp & MY[s], False)
                    hi[c] ^= dp2a(xw & MX[r], yp & MY[s], True)
            lv = (lo[0] & FIELD[0]) | (lo[1] & FIELD[1]) | (lo[2] & FIELD[2])
            hv = (hi[0] & FIELD[0]) | (hi[1] & FIELD[1]) | (hi[2] & FIELD[2])
            return lv ^ (hv << 8)

        L, H, M = leaf_packed(xl, yl), leaf_packed(xh, yh), leaf_packed(xl ^ xh, yl ^ yh)
        got = L ^ ((L ^ H ^ M) << 16) ^ (H << 32)
        assert got == clmul(xa, ya) ^ clmul(xb, yb)


def leaf_merged(pairs) -> int:
    """DotM (csrc/bx_core.cuh: dotm16): the high-byte sums are folded into the
    low-byte accumulators at every step, shifted by 8 -- class c + 1 lands on
    class c, and whatever leaves the 32-bit word is count garbage."""
    acc = [0, 0, 0]
    for xw, yw in pairs:
        yp = byte_perm(yw, 0, 0x3120)
        lo, hi = [0, 0, 0], [0, 0, 0]
        for c in range(3):
            for r in range(3):
                s = (c + 3 - r) % 3
                lo[c] ^= dp2a(xw & MX[r], yp & MY[s], False)
                hi[c] ^= dp2a(xw & MX[r], yp & MY[s], True)
        for c in range(3):
            acc[c] ^= lo[c] ^ ((hi[(c + 1) % 3] << 8) & 0xFFFFFFFF)
    return (acc[0] & FIELD[0]) | (acc[1] & FIELD[1]) | (acc[2] & FIELD[2])


def test_merged_leaf_matches_split_leaf():
    rnd = random.Random(77)
    cases = [[(0xFFFFFFFF, 0xFFFFFFFF)] * 64, [(0xFFFFFFFF, 0xFFFFFFFF)], [(0x80008000, 0x80808080)]]
    cases += [[(rnd.getrandbits(32), rnd.getrandbits(32)) for _ in range(rnd.randint(1, 40))]
              for _ in range(60)]
    for pairs in cases:
        assert leaf_merged(pairs) == want(pairs) & 0xFFFFFFFF
