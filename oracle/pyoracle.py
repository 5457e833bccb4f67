"""Pure-Python restatement of the reference extractor -- TEST INFRASTRUCTURE ONLY.

Small cases only (Python big ints).  Each function cites the reference lines it
restates (reference = /root/reference/pkg/src/blockext, read-only):

* ``gf_mul``      gf2q.py:44-54 (poly_mul), :124-133 (fold table), :156-169 (mul)
* ``ext_ip``      extractor.py:77-87
* ``extract_eq``  extractor.py:182-208 (framing, disjoint q*n-bit windows,
                  LSB-first elements), bitio.py:45-60 and :74-88 (bit order, pad)
* ``pack``        sources.py:116-121
"""
from __future__ import annotations


def modulus_int(exps) -> int:
    v = 0
    for e in exps:
        v |= 1 << e
    return v


def fold_table(q: int, modulus: int) -> list[int]:
    """fold[i] = x^(q+i) mod P (gf2q.py:124-133)."""
    out, t = [], modulus ^ (1 << q)
    for _ in range(q):
        out.append(t)
        t <<= 1
        if t >> q:
            t ^= modulus
    return out


def clmul(a: int, b: int) -> int:
    """Carry-less product, shorter operand drives the loop (gf2q.py:44-54)."""
    if a.bit_length() > b.bit_length():
        a, b = b, a
    r = 0
    while a:
        if a & 1:
            r ^= b
        a >>= 1
        b <<= 1
    return r


def gf_mul(q: int, modulus: int, a: int, b: int, fold=None) -> int:
    """GF(2^q) product (gf2q.py:156-169)."""
    fold = fold or fold_table(q, modulus)
    p = clmul(a, b)
    high, p = p >> q, p & ((1 << q) - 1)
    i = 0
    while high:
        if high & 1:
            p ^= fold[i]
        high >>= 1
        i += 1
    return p


def ext_ip(q: int, modulus: int, xs, ys) -> int:
    """XOR of element products (extractor.py:77-87)."""
    fold = fold_table(q, modulus)
    acc = 0
    for a, b in zip(xs, ys):
        acc ^= gf_mul(q, modulus, a, b, fold)
    return acc


def extract_eq(x: bytes, y: bytes, q: int, n: int, nblocks: int, modulus: int) -> bytes:
    """Packed output of `nblocks` equal-width blocks (extractor.py:182-208, 264-279)."""
    xi = int.from_bytes(x, "little")
    yi = int.from_bytes(y, "little")
    B = q * n
    mask = (1 << q) - 1
    out = 0
    for l in range(nblocks):
        xw = (xi >> (l * B)) & ((1 << B) - 1)
        yw = (yi >> (l * B)) & ((1 << B) - 1)
        xs = [(xw >> (j * q)) & mask for j in range(n)]
        ys = [(yw >> (j * q)) & mask for j in range(n)]
        out |= ext_ip(q, modulus, xs, ys) << (l * q)
    nbits = nblocks * q
    return out.to_bytes((nbits + 7) // 8, "little")


def pack(values, b: int) -> bytes:
    """b-bit samples, LSB-first (sources.py:116-121)."""
    acc = 0
    for i, v in enumerate(values):
        acc |= (int(v) & ((1 << b) - 1)) << (i * b)
    nbits = len(values) * b
    return acc.to_bytes((nbits + 7) // 8, "little")
