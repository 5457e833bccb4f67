"""Helpers shared by the test modules (not a package; imported by name)."""
import io
from fractions import Fraction

import numpy as np


def case_inputs(c):
    rng = np.random.default_rng(c["seed"])
    return rng.bytes(c["x_len"]), rng.bytes(c["y_len"])


def tiny_eq_plan(bx, b, samples, rate, vec_len, field_bits):
    """Hand-assembled plan like the reference tests' tiny_eq_plan
    (pkg/tests/test_extractor.py:32-38)."""
    rate = bx.params.as_rational(rate)
    nb = samples * b // (field_bits * vec_len)
    draft = bx.EqPlan(b, samples, rate, Fraction(1, 2), vec_len, field_bits, nb, nb * field_bits, 0.0)
    return bx.EqPlan(**{**draft.__dict__, "log2_error": bx.error_bound_eq(draft)})


def report_dict(rep):
    return {
        "mode": rep.mode, "blocks_completed": rep.blocks_completed,
        "x_bits_consumed": rep.x_bits_consumed, "y_bits_consumed": rep.y_bits_consumed,
        "output_bits": rep.output_bits, "x_discarded_tail_bits": rep.x_discarded_tail_bits,
        "y_discarded_tail_bits": rep.y_discarded_tail_bits,
        "log2_error_bound": repr(rep.log2_error_bound), "stop_reason": rep.stop_reason,
        "pad_bits": rep.pad_bits,
    }


class DribbleIO:
    """File-like object returning at most `step` bytes per read (reference
    pkg/tests/test_bitio.py:11-19 pattern)."""

    def __init__(self, data: bytes, step: int = 1):
        self._buf = io.BytesIO(data)
        self._step = step

    def read(self, size: int) -> bytes:
        return self._buf.read(min(size, self._step))


def place(z: bytes, out):
    """Stand-in compute helper: like sharding.extract_packed(out=...), write the
    packed bytes into `out` (a CPU uint8 tensor) when given and return a view."""
    if out is None:
        return z
    import numpy as np
    arr = out.numpy()
    arr[:len(z)] = np.frombuffer(z, dtype=np.uint8)
    return arr[:len(z)]
