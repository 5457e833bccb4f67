"""Plans and log2-domain error bounds (host math, no GPU work).

Mirrors the planning API of the reference (pkg/src/blockext/params.py) so a
user's plans carry over unchanged:

* ``EqPlan`` / ``NeqPlan`` fields           params.py:91-132
* ``plan_eq``  (n = ceil(24/(2r-1)), q steps by b)   params.py:135-198
* ``plan_neq`` (closed-form start width)    params.py:201-258
* ``error_bound_block/eq/neq``              params.py:263-327

The bounds are evaluated in double precision in the same operation order as the
reference, so reports compare equal float-for-float.
"""
from __future__ import annotations

import functools
import math
from dataclasses import dataclass
from fractions import Fraction

from .errors import CapacityError, DivergenceError, UnsupportedRateError

LOG2_SQRT3 = 0.5 * math.log2(3.0)
MAX_SAMPLE_BITS = 64
MAX_FIELD_BITS = 128


def _log2_big(v: int) -> float:
    if v <= 0:
        raise ValueError("log2 of non-positive integer")
    drop = v.bit_length() - 900
    if drop <= 0:
        return math.log2(v)
    return math.log2(v >> drop) + drop


def log2_fraction(fr: Fraction) -> float:
    if fr <= 0:
        raise ValueError("log2 of non-positive value")
    return _log2_big(fr.numerator) - _log2_big(fr.denominator)


def as_rational(value, name: str = "value") -> Fraction:
    """Exact rational from a Fraction, int or string ("3/4", "0.75", "2^-30")."""
    if isinstance(value, bool):
        raise TypeError(f"{name} must be rational, got bool")
    if isinstance(value, Fraction):
        return value
    if isinstance(value, int):
        return Fraction(value)
    if isinstance(value, float):
        raise TypeError(f"{name} must be an exact rational (Fraction, int, or string); "
                        "floats near a ceiling boundary can change derived parameters")
    if isinstance(value, str):
        s = value.strip()
        if "/" in s:
            top, bottom = s.split("/", 1)
            return as_rational(top.strip(), name) / as_rational(bottom.strip(), name)
        if "^" in s:
            base, exp = s.split("^", 1)
            return Fraction(int(base)) ** int(exp)
        return Fraction(s)
    raise TypeError(f"cannot interpret {name}={value!r} as a rational")


def parse_count(text: str) -> int:
    s = text.strip()
    if "^" in s:
        base, exp = s.split("^", 1)
        v = int(base) ** int(exp)
    else:
        v = int(s)
    if v <= 0:
        raise ValueError(f"count must be positive, got {text!r}")
    return v


def parse_probability(text: str) -> Fraction:
    return as_rational(text, "probability")


@dataclass(frozen=True)
class EqPlan:
    """Equal-block plan: the fields the engine reads (reference params.py:91-108)."""

    bits_per_sample: int
    num_samples: int
    entropy_rate: Fraction
    epsilon: Fraction
    vec_len: int
    field_bits: int
    num_blocks: int
    output_bits: int
    log2_error: float

    @property
    def block_bits(self) -> int:
        return self.field_bits * self.vec_len


@dataclass(frozen=True)
class NeqPlan:
    """Incremental-block plan (reference params.py:111-132)."""

    bits_per_sample: int
    entropy_rate: Fraction
    vec_len: int
    first_field_bits: int
    growth: int
    log2_error_limit: float | None

    def field_bits_for_block(self, index: int) -> int:
        if index < 1:
            raise ValueError("block index is 1-based")
        return self.first_field_bits + (index - 1) * self.growth * self.bits_per_sample

    def output_bits_after(self, k: int) -> int:
        if k < 0:
            raise ValueError("block count must be >= 0")
        step = self.growth * self.bits_per_sample
        return k * self.first_field_bits + (k - 1) * k * step // 2


def vec_len_for_rate(rate: Fraction) -> int:
    """n = ceil(24 / (2*rate - 1)), exactly."""
    return math.ceil(Fraction(24) / (2 * rate - 1))


def _check_rate(rate: Fraction) -> None:
    if rate <= Fraction(1, 2):
        raise UnsupportedRateError(
            f"min-entropy rate {rate} <= 1/2; extraction requires rate > 1/2")
    if rate > 1:
        raise ValueError(f"min-entropy rate {rate} exceeds 1")


def _check_b(b: int) -> None:
    if not 1 <= b <= MAX_SAMPLE_BITS:
        raise ValueError(f"bits per sample must be in 1..{MAX_SAMPLE_BITS}")


def error_bound_block(vec_len: int, field_bits: int, entropy_rate) -> float:
    """log2(sqrt 3) - 1/4 - (rate/4 - 1/8)*q*n + 2q, fixed evaluation order."""
    if isinstance(entropy_rate, Fraction):
        # the hashable common case: memoised (a streaming caller evaluates the
        # same plan's bound once per call)
        return _error_bound_block_cached(vec_len, field_bits, entropy_rate)
    return _error_bound_block(vec_len, field_bits, entropy_rate)


@functools.lru_cache(maxsize=256)
def _error_bound_block_cached(vec_len: int, field_bits: int, entropy_rate: Fraction) -> float:
    return _error_bound_block(vec_len, field_bits, entropy_rate)


def _error_bound_block(vec_len: int, field_bits: int, entropy_rate) -> float:
    rate = as_rational(entropy_rate, "entropy_rate")
    if vec_len < 1 or field_bits < 1:
        raise ValueError("vec_len and field_bits must be >= 1")
    if not Fraction(1, 2) < rate <= 1:
        raise ValueError(f"entropy rate {rate} outside (1/2, 1]")
    slope = float(rate / 4 - Fraction(1, 8))
    return LOG2_SQRT3 - 0.25 - slope * (field_bits * vec_len) + 2.0 * field_bits


def _total_bound(num_blocks: int, n: int, q: int, rate: Fraction) -> float:
    if num_blocks == 0:
        return float("-inf")
    return _log2_big(num_blocks) + error_bound_block(n, q, rate)


def error_bound_eq(plan, blocks: int | None = None) -> float:
    if blocks is None:
        blocks = plan.num_blocks
    if blocks < 0:
        raise ValueError("block count must be >= 0")
    return _total_bound(blocks, plan.vec_len, plan.field_bits, plan.entropy_rate)


def _geometric_limit(q1: int, step_bits: int) -> float:
    if step_bits < 1:
        raise DivergenceError("error series converges only for growth >= 1")
    return LOG2_SQRT3 - 0.25 - q1 - math.log2(1.0 - 2.0 ** (-step_bits))


def error_bound_neq(plan, k: int | None = None) -> float:
    if k is None:
        if plan.growth < 1:
            raise DivergenceError(
                "growth = 0 repeats one block width forever; the error series diverges")
        return _geometric_limit(plan.first_field_bits, plan.growth * plan.bits_per_sample)
    if k < 1:
        raise ValueError("block count must be >= 1")
    terms = [error_bound_block(plan.vec_len, plan.field_bits_for_block(i), plan.entropy_rate)
             for i in range(1, k + 1)]
    anchor = terms[0]
    total = 0.0
    for t in terms:
        total += 2.0 ** (t - anchor)
    return anchor + math.log2(total)


def plan_eq(bits_per_sample: int, num_samples: int, entropy_rate, epsilon) -> EqPlan:
    rate = as_rational(entropy_rate, "entropy_rate")
    eps = as_rational(epsilon, "epsilon")
    _check_rate(rate)
    _check_b(bits_per_sample)
    if not 0 < eps < 1:
        raise ValueError(f"epsilon must be in (0,1), got {eps}")
    if num_samples < 1:
        raise ValueError("sample count must be positive")
    b = bits_per_sample
    n = vec_len_for_rate(rate)
    need = Fraction(num_samples) / (eps * n)
    q = b
    while (1 << q) < need:
        q += b
    target = log2_fraction(eps)
    while True:
        if q > MAX_FIELD_BITS:
            raise CapacityError(
                f"derived field width {q} exceeds the {MAX_FIELD_BITS}-bit implementation cap")
        blocks = num_samples * b // (q * n)
        bound = _total_bound(blocks, n, q, rate)
        if bound <= target:
            break
        q += b
    return EqPlan(b, num_samples, rate, eps, n, q, blocks, blocks * q, bound)


def plan_neq(bits_per_sample: int, entropy_rate, first_field_bits: int | None = None,
             growth: int = 1, epsilon=None) -> NeqPlan:
    rate = as_rational(entropy_rate, "entropy_rate")
    _check_rate(rate)
    _check_b(bits_per_sample)
    if growth < 0:
        raise ValueError("growth must be >= 0")
    b = bits_per_sample
    n = vec_len_for_rate(rate)
    if first_field_bits is None:
        if epsilon is None:
            raise ValueError("need first_field_bits or epsilon")
        if growth < 1:
            raise DivergenceError("infinite-run planning requires growth >= 1")
        eps = as_rational(epsilon, "epsilon")
        if not 0 < eps < 1:
            raise ValueError(f"epsilon must be in (0,1), got {eps}")
        target = log2_fraction(eps)
        q1 = b
        while _geometric_limit(q1, growth * b) > target:
            q1 += b
            if q1 > MAX_FIELD_BITS:
                raise CapacityError(f"starting width needed for epsilon={eps} exceeds "
                                    f"the {MAX_FIELD_BITS}-bit cap")
    else:
        q1 = first_field_bits
        if q1 < 1 or q1 % b:
            raise ValueError(f"starting width {q1} must be a positive multiple of b={b}")
        if q1 > MAX_FIELD_BITS:
            raise CapacityError(
                f"starting width {q1} exceeds the {MAX_FIELD_BITS}-bit implementation cap")
    limit = _geometric_limit(q1, growth * b) if growth >= 1 else None
    return NeqPlan(b, rate, n, q1, growth, limit)


def extraction_rate(plan) -> tuple[float, float]:
    rate = plan.entropy_rate
    exact = Fraction(1) / (2 * rate * plan.vec_len)
    approx = (2 * rate - 1) / (48 * rate)
    return float(exact), float(approx)


def is_eq_plan(plan) -> bool:
    """Duck typing: the equal-block engine reads field_bits and num_blocks."""
    return hasattr(plan, "field_bits") and hasattr(plan, "num_blocks")


def is_neq_plan(plan) -> bool:
    return hasattr(plan, "first_field_bits") and hasattr(plan, "growth")


__all__ = [
    "EqPlan", "NeqPlan", "LOG2_SQRT3", "MAX_SAMPLE_BITS", "as_rational",
    "error_bound_block", "error_bound_eq", "error_bound_neq", "extraction_rate",
    "log2_fraction", "parse_count", "parse_probability", "plan_eq", "plan_neq",
]
