"""Exhaustive verification suites on the GPU.

Same functions, reports and limits as the reference's brute-force oracles
(pkg/src/blockext/verify.py).  The exhaustive part -- every inner product
<x, y> of an instance with t = q*n <= 16 input bits per source -- runs on the
sm_100a kernels (``bx_ip_table``, ``bx_ip_histograms``, ``bx_rows_uniform``);
the reductions over those tables (Gram matrices, Walsh spectra, weighted
histograms) run as device tensor operations.  Small host-side tables
(shift tables, first-bit rows, parity) and the q <= 4 / q <= 8 checks
(XOR lemma, functional bijection) are exact integer host math.

* ``check_hadamard``      reference verify.py:212-297 (direct Gram / counts)
* ``check_one_bit_bias``  verify.py:316-366
* ``check_extractor_distance``  verify.py:384-422
* ``check_xor_lemma_instance``  verify.py:427-460
* ``check_first_bit_bijection`` verify.py:465-488
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from itertools import combinations
from typing import Sequence

import numpy as np

from .errors import InfeasibleError
from .gf2q import GFContext
from .params import LOG2_SQRT3

MAX_HADAMARD_BITS = 16
MAX_DENSE_BITS = 12
DIRECT_METHOD_BITS = 8
HIST_BATCH = 4096


# ------------------------------------------------------------ host tables

def shift_tables(ctx: GFContext) -> list[np.ndarray]:
    """T[j][v] = v * x^j mod modulus for all q-bit v (q <= 16)."""
    q = ctx.q
    if q > 16:
        raise InfeasibleError("shift tables limited to q <= 16")
    t = np.arange(1 << q, dtype=np.uint32)
    out = []
    for _ in range(q):
        out.append(t.copy())
        t = t << np.uint32(1)
        high = (t >> np.uint32(q)) & np.uint32(1)
        t ^= high * np.uint32(ctx.modulus)
    return out


def first_bit_rows(ctx: GFContext) -> np.ndarray:
    """brow[v]: bit j = first bit of v * x^j, so first_bit(a*v) = parity(a & brow[v])."""
    brow = np.zeros(1 << ctx.q, dtype=np.uint32)
    for j, tab in enumerate(shift_tables(ctx)):
        brow |= (tab & np.uint32(1)) << np.uint32(j)
    return brow


def parity_table(q: int) -> np.ndarray:
    v = np.arange(1 << q, dtype=np.uint32)
    p = v.copy()
    s = 1
    while s < 32:
        p ^= p >> np.uint32(s)
        s <<= 1
    return (p & np.uint32(1)).astype(np.uint8)


_parity_table = parity_table   # reference-internal name (verify.py:252-259)


def _window_table(ctx: GFContext, base: int, width: int) -> np.ndarray:
    """W[d, u] = d * (u << base) mod modulus for all q-bit d and width-bit u
    (reference-internal helper, verify.py:166-182): XOR of shift-table columns
    per set bit of u."""
    tabs = shift_tables(ctx)
    us = np.arange(1 << width)
    w = np.zeros((1 << ctx.q, 1 << width), dtype=np.uint32)
    for j in range(width):
        w[:, ((us >> j) & 1).astype(bool)] ^= tabs[base + j][:, None]
    return w


def walsh_transform(rows) -> np.ndarray:
    """out[..., a] = sum_w rows[..., w] * (-1)^popcount(a & w), exact int64."""
    a = np.array(rows, dtype=np.int64, copy=True)
    n = a.shape[-1]
    if n & (n - 1):
        raise ValueError("length must be a power of two")
    h = 1
    while h < n:
        b = a.reshape(a.shape[:-1] + (n // (2 * h), 2, h))
        a = np.stack((b[..., 0, :] + b[..., 1, :], b[..., 0, :] - b[..., 1, :]), axis=-2).reshape(a.shape)
        h *= 2
    return a


def _walsh_torch(t):
    """Walsh transform along the last axis of a torch tensor (float64/int64)."""
    n = t.shape[-1]
    h = 1
    while h < n:
        b = t.reshape(t.shape[:-1] + (n // (2 * h), 2, h))
        t = torch_stack((b[..., 0, :] + b[..., 1, :], b[..., 0, :] - b[..., 1, :]), -2).reshape(t.shape)
        h *= 2
    return t


def torch_stack(ts, dim):
    import torch
    return torch.stack(ts, dim=dim)


def _feasible(ctx: GFContext, n: int, cap: int, what: str) -> int:
    t = ctx.q * n
    if n < 1:
        raise ValueError("n must be >= 1")
    if t > cap:
        raise InfeasibleError(f"{what} limited to q*n <= {cap}, got {t}")
    return t


def _default_modulus(ctx: GFContext) -> None:
    if not ctx._default:
        raise NotImplementedError("the exhaustive verification kernels use the shipped default modulus")


# ---------------------------------------------------------- device tables

def ip_value_table_device(ctx: GFContext, n: int, device=None):
    """(2^t, 2^t) int64 CUDA tensor of <x, y> (t = q*n <= 12)."""
    import torch

    from . import _lib
    from . import device as D

    t = _feasible(ctx, n, MAX_DENSE_BITS, "dense inner-product table")
    _default_modulus(ctx)
    dev = D.require_cuda(device)
    size = 1 << t
    z = torch.empty(size * size, dtype=torch.int16, device=dev)
    with torch.cuda.device(dev):
        _lib.check(_lib.lib().bx_ip_table(ctx.q, n, 0, size, z.data_ptr(), D.stream_ptr(None, dev)),
                   "bx_ip_table")
    return z.view(size, size).to(torch.int64) & ((1 << 16) - 1)


def ip_value_table(ctx: GFContext, n: int) -> np.ndarray:
    """Dense table of <x, y> for all x, y (reference verify.py:200-207), computed
    on the GPU; returned on the host as uint16."""
    return ip_value_table_device(ctx, n).cpu().numpy().astype(np.uint16)


# ------------------------------------------------------ hadamard property

def check_hadamard(ctx: GFContext, n: int, method: str = "auto") -> bool:
    """Whether every f_a(x, y) = first bit of a*<x, y> has exactly
    uncorrelated rows (zero tolerance)."""
    t = _feasible(ctx, n, MAX_HADAMARD_BITS, "hadamard check")
    if method == "auto":
        method = "direct" if t <= DIRECT_METHOD_BITS else "counts"
    if method == "direct":
        return _hadamard_direct(ctx, n)
    if method == "counts":
        return _hadamard_counts(ctx, n)
    raise ValueError(f"unknown method {method!r}")


def _hadamard_direct(ctx: GFContext, n: int) -> bool:
    """Literal Gram matrix of every f_a's +/-1 row matrix (t <= 12)."""
    import torch

    t = ctx.q * n
    if t > MAX_DENSE_BITS:
        raise InfeasibleError(f"direct method needs q*n <= {MAX_DENSE_BITS}")
    size = 1 << t
    z = ip_value_table_device(ctx, n)
    dev = z.device
    brow = torch.from_numpy(first_bit_rows(ctx).astype(np.int64)).to(dev)
    par = torch.from_numpy(parity_table(ctx.q).astype(np.int64)).to(dev)
    bz = brow[z]                                        # (size, size)
    eye = size * torch.eye(size, dtype=torch.float64, device=dev)
    for a in range(1, 1 << ctx.q):
        fa = par[a & bz]
        signs = (1 - 2 * fa).to(torch.float64)
        gram = signs @ signs.T
        if not torch.equal(gram, eye):
            return False
    return True


def _hadamard_counts(ctx: GFContext, n: int) -> bool:
    """Histogram form (reference verify.py:262-297): for every nonzero
    difference d the pair sums are sum_v counts_d[v] (-1)^(first bit of a*v);
    uniform histograms reduce to the functional balances."""
    import torch

    from . import _lib
    from . import device as D

    _default_modulus(ctx)
    q = ctx.q
    t = q * n
    bins = 1 << q
    brow = first_bit_rows(ctx)
    hist = np.bincount(brow, minlength=bins)
    balances_ok = not np.any(walsh_transform(hist)[1:])
    expected = 1 << (t - q)
    dev = D.require_cuda()
    L = _lib.lib()
    total = (1 << t) - 1
    batch = max(1, min(HIST_BATCH, (1 << 26) // bins))
    counts = torch.empty(batch * bins, dtype=torch.int32, device=dev)
    flags = torch.empty(batch, dtype=torch.uint8, device=dev)
    sp = D.stream_ptr(None, dev)
    d = 1
    while d <= total:
        nd = min(batch, total - d + 1)
        with torch.cuda.device(dev):
            _lib.check(L.bx_ip_histograms(q, n, d, nd, counts.data_ptr(), sp), "bx_ip_histograms")
            _lib.check(L.bx_rows_uniform(counts.data_ptr(), nd, bins, expected, flags.data_ptr(), sp),
                       "bx_rows_uniform")
        uni = flags[:nd].cpu().numpy().astype(bool)
        if uni.all():
            if not balances_ok:
                return False
        else:
            if not balances_ok and uni.any():
                return False
            rows = counts[:nd * bins].view(nd, bins).cpu().numpy().astype(np.int64)
            for r in np.nonzero(~uni)[0]:
                grouped = np.bincount(brow, weights=rows[r].astype(np.float64), minlength=bins)
                if np.any(walsh_transform(np.rint(grouped).astype(np.int64))[1:]):
                    return False
        d += nd
    return True


def hadamard_instances(max_bits: int = MAX_HADAMARD_BITS):
    """All (q, n) with q * n <= max_bits, in the reference's sweep order."""
    for q in range(1, max_bits + 1):
        for n in range(1, max_bits // q + 1):
            yield q, n


# ------------------------------------------------- one-bit bias, flat sources

@dataclass(frozen=True)
class BiasReport:
    input_bits: int
    entropy_floor: int
    max_bias: float
    bound: float
    pairs_tested: int
    exhaustive: bool

    @property
    def holds(self) -> bool:
        return self.max_bias <= self.bound + 1e-12


def check_one_bit_bias(ctx: GFContext, n: int, k: int, *, seed: int = 0,
                       sampled_pairs: int = 200, exhaustive_limit: int = 10**5) -> BiasReport:
    """Max bias of every f_a over pairs of flat sources with min-entropy k
    (reference verify.py:316-366); the support pairs are evaluated in batches
    on the device (gather, one-hot histogram, Walsh spectrum)."""
    import torch

    t = _feasible(ctx, n, MAX_DENSE_BITS, "one-bit bias check")
    if not 0 <= k <= t:
        raise ValueError(f"entropy floor k={k} outside 0..{t}")
    size, support = 1 << t, 1 << k
    z = ip_value_table_device(ctx, n)
    dev = z.device
    brow = torch.from_numpy(first_bit_rows(ctx).astype(np.int64)).to(dev)
    w_of_z = brow[z]
    n_subsets = math.comb(size, support)
    exhaustive = n_subsets <= exhaustive_limit and n_subsets**2 <= exhaustive_limit
    if exhaustive:
        subsets = [np.fromiter(c, dtype=np.int64) for c in combinations(range(size), support)]
        pairs = [(sx, sy) for sx in subsets for sy in subsets]
    else:
        rng = np.random.default_rng(seed)
        pairs = [(rng.choice(size, size=support, replace=False).astype(np.int64),
                  rng.choice(size, size=support, replace=False).astype(np.int64))
                 for _ in range(sampled_pairs)]
    bins = 1 << ctx.q
    denom = float(support) * float(support)
    max_bias = 0.0
    chunk = max(1, (1 << 22) // (support * support + bins))
    for s in range(0, len(pairs), chunk):
        part = pairs[s:s + chunk]
        sx = torch.from_numpy(np.stack([p[0] for p in part])).to(dev)
        sy = torch.from_numpy(np.stack([p[1] for p in part])).to(dev)
        cells = w_of_z[sx[:, :, None], sy[:, None, :]].reshape(len(part), -1)
        grouped = torch.zeros(len(part), bins, dtype=torch.int64, device=dev)
        grouped.scatter_add_(1, cells, torch.ones_like(cells))
        spectrum = _walsh_torch(grouped)
        bias = float(spectrum[:, 1:].abs().max().item()) / denom if bins > 1 else 0.0
        max_bias = max(max_bias, bias)
    bound = 2.0 ** (1.0 - (2 * k - t) / 2.0)
    return BiasReport(t, k, max_bias, bound, len(pairs), exhaustive)


# ---------------------------------------------------- exact output distance

@dataclass(frozen=True)
class DistanceReport:
    description: str
    input_bits: int
    rate: float
    distance: float
    bound: float

    @property
    def holds(self) -> bool:
        return self.distance <= self.bound + 1e-12


def check_extractor_distance(ctx: GFContext, n: int, px: Sequence[float], py: Sequence[float],
                             declared_rate: float | None = None,
                             description: str = "") -> DistanceReport:
    """Exact total-variation distance of <X, Y> from uniform for explicit
    source distributions (reference verify.py:384-422)."""
    import torch

    t = _feasible(ctx, n, MAX_DENSE_BITS, "distance check")
    size = 1 << t
    px = np.asarray(px, dtype=np.float64)
    py = np.asarray(py, dtype=np.float64)
    for name, p in (("px", px), ("py", py)):
        if p.shape != (size,):
            raise ValueError(f"{name} must have {size} entries")
        if np.any(p < 0) or abs(float(p.sum()) - 1.0) > 2.0 ** -30:
            raise ValueError(f"{name} is not a probability distribution")
    hmin = min(-math.log2(float(px.max())), -math.log2(float(py.max())))
    if declared_rate is None:
        rate = hmin / t
    else:
        rate = declared_rate
        if hmin + 1e-12 < rate * t:
            raise ValueError(f"tables have min-entropy {hmin:.6f} < declared rate * qn = {rate * t:.6f}")
    z = ip_value_table_device(ctx, n)
    dev = z.device
    w = torch.outer(torch.from_numpy(px).to(dev), torch.from_numpy(py).to(dev))
    out = torch.zeros(1 << ctx.q, dtype=torch.float64, device=dev)
    out.scatter_add_(0, z.reshape(-1), w.reshape(-1))
    distance = 0.5 * float((out - 1.0 / (1 << ctx.q)).abs().sum().item())
    log2_bound = LOG2_SQRT3 - 0.25 - (rate / 4.0 - 0.125) * t + 2.0 * ctx.q
    return DistanceReport(description or f"q={ctx.q} n={n}", t, rate, distance,
                          min(1.0, 2.0 ** log2_bound))


# ------------------------------------------------------------- XOR lemma

def xor_lemma_sides(q: int, joint) -> tuple[float, float]:
    """(lhs, rhs) of the XOR lemma with classical side information (q <= 4)."""
    if q > 4:
        raise InfeasibleError("XOR lemma check limited to q <= 4")
    joint = np.asarray(joint, dtype=np.float64)
    if joint.ndim != 2 or joint.shape[0] != 1 << q:
        raise ValueError(f"joint must be (2^{q}, num_e)")
    if joint.shape[1] > 16:
        raise InfeasibleError("classical side information limited to <= 16 values")
    if np.any(joint < 0) or abs(float(joint.sum()) - 1.0) > 2.0 ** -30:
        raise ValueError("joint is not a probability distribution")
    pe = joint.sum(axis=0)
    lhs = float(np.abs(joint - pe[None, :] / (1 << q)).sum())
    par = parity_table(q)
    zs = np.arange(1 << q)
    rhs = 0.0
    for s in range(1, 1 << q):
        bits = par[s & zs]
        p1 = joint[bits == 1].sum(axis=0)
        p0 = joint[bits == 0].sum(axis=0)
        rhs += float(np.abs(p1 - pe / 2).sum() + np.abs(p0 - pe / 2).sum())
    return lhs, rhs * float(1 << q)


def check_xor_lemma_instance(q: int, joint) -> bool:
    lhs, rhs = xor_lemma_sides(q, joint)
    return lhs <= rhs + 1e-12


# ---------------------------------------------- S <-> a functional bijection

def check_first_bit_bijection(ctx: GFContext) -> bool:
    """Each parity functional S.z equals first_bit(a*z) for exactly one a (q <= 8)."""
    if ctx.q > 8:
        raise InfeasibleError("bijection check limited to q <= 8")
    q = ctx.q
    par = parity_table(q)
    zs = np.arange(1 << q)
    brow = first_bit_rows(ctx)
    seen = {}
    for a in range(1 << q):
        key = par[a & brow[zs]].tobytes()
        if key in seen:
            return False
        seen[key] = a
    for s in range(1 << q):
        key = par[s & zs].astype(np.uint8).tobytes()
        if key not in seen or (s == 0) != (seen[key] == 0):
            return False
    return True


__all__ = ["BiasReport", "DistanceReport", "MAX_DENSE_BITS", "MAX_HADAMARD_BITS",
           "check_extractor_distance", "check_first_bit_bijection", "check_hadamard",
           "check_one_bit_bias", "check_xor_lemma_instance", "first_bit_rows",
           "hadamard_instances", "ip_value_table", "shift_tables", "walsh_transform",
           "xor_lemma_sides"]
