"""Generate the golden fixtures by running the REFERENCE implementation.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports the reference package ``blockext`` from /root/reference/pkg/src and
records its outputs for seeded inputs.  The fixtures (JSON + one small binary)
are committed; nothing on the GPU box reads /root/reference.

Fixtures:
  moduli.json     the reference modulus table (_moduli.py:13-142)
  gf_mul.json     GFContext.mul KATs for every q = 1..128 (gf2q.py:156-169)
  ext_ip.json     ext_ip KATs (extractor.py:77-87)
  eq_cases.json   extract_eq(...).run(sink) outputs + reports: every q = 1..128,
                  odd shapes, short / unequal streams, max_blocks, completed runs
  neq_cases.json  extract_neq outputs + reports (growth 0..3, width cap)
  pack.json       _pack_samples for b = 1..64 (sources.py:116-121)
  c1.json + c1_out.bin   config 1 in full (2 x 2^20 bits, q=32, n=4)
  sampled.json    single-block outputs at sampled block indices of the full-size
                  configs (windows regenerated with PCG64 advance)
  streams.json    sha256 of stream prefixes from the reference generate(), pinning
                  paper_2402_14607_b200.workloads against it
  markov.json     generate(markov(T, b, seed), count) outputs (sources.py:141-152)
  verify.json     verification-suite results: ip_value_table hashes, one-bit bias
                  and exact-distance reports, hadamard verdicts (verify.py)
"""
from __future__ import annotations

import hashlib
import io
import json
import pathlib
import random
import sys
from fractions import Fraction

import numpy as np

HERE = pathlib.Path(__file__).resolve().parent
REPO = HERE.parents[1]
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(REPO))

import blockext  # noqa: E402  (the reference)
from blockext import extractor as R_ext  # noqa: E402
from blockext import gf2q as R_gf  # noqa: E402
from blockext import params as R_params  # noqa: E402
from blockext import sources as R_src  # noqa: E402
from blockext._moduli import MODULUS_EXPONENTS  # noqa: E402

from paper_2402_14607_b200 import workloads as W  # noqa: E402


def h(v: int) -> str:
    return format(v, "x")


def tiny_plan(b, samples, rate, n, q):
    rate = R_params.as_rational(rate)
    nb = samples * b // (q * n)
    draft = R_params.EqPlan(b, samples, rate, Fraction(1, 2), n, q, nb, nb * q, 0.0)
    return R_params.EqPlan(**{**draft.__dict__, "log2_error": R_params.error_bound_eq(draft)})


def report_dict(rep) -> dict:
    return {
        "mode": rep.mode, "blocks_completed": rep.blocks_completed,
        "x_bits_consumed": rep.x_bits_consumed, "y_bits_consumed": rep.y_bits_consumed,
        "output_bits": rep.output_bits, "x_discarded_tail_bits": rep.x_discarded_tail_bits,
        "y_discarded_tail_bits": rep.y_discarded_tail_bits,
        "log2_error_bound": repr(rep.log2_error_bound), "stop_reason": rep.stop_reason,
        "pad_bits": rep.pad_bits,
    }


def dump(name: str, obj) -> None:
    (HERE / name).write_text(json.dumps(obj, indent=None, separators=(",", ":")) + "\n")
    print(f"wrote {name}", file=sys.stderr)


def make_moduli():
    dump("moduli.json", {str(q): list(e) for q, e in MODULUS_EXPONENTS.items()})


def make_gf():
    out = {}
    for q in range(1, 129):
        rnd = random.Random(7000 + q)
        ctx = R_gf.field(q)
        vals = [(0, ctx.mask), (1, ctx.mask), (ctx.mask, ctx.mask)]
        vals += [(rnd.getrandbits(q), rnd.getrandbits(q)) for _ in range(6)]
        out[str(q)] = [[h(a), h(b), h(ctx.mul(a, b))] for a, b in vals]
    dump("gf_mul.json", out)


def make_ext_ip():
    rnd = random.Random(11)
    cases = []
    for q, n in [(1, 1), (1, 2), (2, 3), (4, 64), (8, 5), (13, 7), (32, 4), (56, 48),
                 (58, 120), (64, 3), (80, 71), (100, 9), (127, 4), (128, 8)]:
        ctx = R_gf.field(q)
        xs = [rnd.getrandbits(q) for _ in range(n)]
        ys = [rnd.getrandbits(q) for _ in range(n)]
        cases.append({"q": q, "x": [h(v) for v in xs], "y": [h(v) for v in ys],
                      "z": h(R_ext.ext_ip(ctx, xs, ys))})
    dump("ext_ip.json", cases)


def run_eq(case):
    rng = np.random.default_rng(case["seed"])
    xb = rng.bytes(case["x_len"])
    yb = rng.bytes(case["y_len"])
    plan = tiny_plan(case["b"], case["samples"], case.get("rate", "3/4"), case["n"], case["q"])
    sink = io.BytesIO()
    rep = R_ext.extract_eq(xb, yb, plan, max_blocks=case.get("max_blocks")).run(sink)
    case = dict(case)
    case["out"] = sink.getvalue().hex()
    case["report"] = report_dict(rep)
    case["plan_log2_error"] = repr(plan.log2_error)
    return case


def make_eq_cases():
    rnd = random.Random(20251020)
    cases = []
    seed = 1000
    # every field width, random vector length and block count
    for q in range(1, 129):
        n = rnd.randint(1, 12)
        blocks = rnd.randint(1, 24)
        samples = blocks * q * n
        nbytes = (samples + 7) // 8
        cases.append({"tag": f"q{q}", "q": q, "n": n, "b": 1, "samples": samples,
                      "x_len": nbytes, "y_len": nbytes, "seed": seed})
        seed += 1
    # benchmark shapes and alignment stress shapes
    for q, n, blocks in [(4, 64, 300), (4, 128, 150), (2, 64, 400), (8, 64, 200),
                         (16, 64, 100), (32, 64, 60), (32, 4, 700), (128, 8, 80),
                         (56, 48, 12), (58, 120, 6), (80, 71, 7), (13, 7, 90),
                         (1, 24, 160), (3, 50, 40), (127, 3, 33), (96, 5, 21),
                         (64, 16, 40), (17, 33, 19), (33, 17, 23)]:
        samples = blocks * q * n
        nbytes = (samples + 7) // 8
        cases.append({"tag": f"shape_q{q}_n{n}", "q": q, "n": n, "b": 1, "samples": samples,
                      "x_len": nbytes, "y_len": nbytes, "seed": seed})
        seed += 1
    # report semantics: remainder, exhaustion, unequal lengths, max_blocks, b>1
    specials = [
        {"tag": "completed_remainder", "q": 8, "n": 6, "b": 8, "samples": 100,
         "x_len": 100, "y_len": 100},
        {"tag": "x_short", "q": 8, "n": 5, "b": 8, "samples": 100, "x_len": 43, "y_len": 100},
        {"tag": "y_short", "q": 8, "n": 5, "b": 8, "samples": 100, "x_len": 100, "y_len": 43},
        {"tag": "long_tail_70k", "q": 8, "n": 5, "b": 8, "samples": 200_000,
         "x_len": 1000, "y_len": 70_000},
        {"tag": "long_tail_200k", "q": 16, "n": 48, "b": 8, "samples": 400_000,
         "x_len": 70_001, "y_len": 200_000},
        {"tag": "block_limit", "q": 16, "n": 4, "b": 16, "samples": 4000,
         "x_len": 8000, "y_len": 8000, "max_blocks": 37},
        {"tag": "max_beyond_plan", "q": 12, "n": 4, "b": 4, "samples": 960,
         "x_len": 480, "y_len": 480, "max_blocks": 10_000},
        {"tag": "empty", "q": 8, "n": 5, "b": 8, "samples": 100, "x_len": 0, "y_len": 0},
        {"tag": "one_block", "q": 80, "n": 71, "b": 16, "samples": 355,
         "x_len": 710, "y_len": 710},
        {"tag": "width_cap_eq", "q": 129, "n": 2, "b": 1, "samples": 1000,
         "x_len": 125, "y_len": 125},
        {"tag": "big_b", "q": 64, "n": 3, "b": 64, "samples": 30, "x_len": 240, "y_len": 240},
        {"tag": "multi_fill", "q": 32, "n": 4, "b": 8, "samples": 300_000,
         "x_len": 300_000, "y_len": 300_000},
    ]
    for s in specials:
        s["seed"] = seed
        seed += 1
        cases.append(s)
    dump("eq_cases.json", [run_eq(c) for c in cases])


def make_neq_cases():
    rnd = random.Random(777)
    cases = []
    for i in range(40):
        b = rnd.choice([1, 2, 4, 8, 16])
        growth = rnd.randint(0, 3)
        q1 = b * rnd.randint(1, max(1, 32 // b))
        k = rnd.randint(1, 9)
        plan = R_params.plan_neq(b, "3/4", q1, growth)
        need = sum(min(plan.field_bits_for_block(j), 128) * plan.vec_len for j in range(1, k + 1))
        nbytes = (need + 7) // 8 + rnd.randint(0, 40)
        cases.append({"b": b, "growth": growth, "q1": q1, "max_blocks": rnd.choice([k, None]),
                      "x_len": nbytes, "y_len": nbytes - rnd.randint(0, 3), "seed": 5000 + i})
    cases.append({"b": 16, "growth": 1, "q1": 16, "max_blocks": None, "x_len": 200_000,
                  "y_len": 200_000, "seed": 0, "zeros": True})
    cases.append({"b": 8, "growth": 1, "q1": 8, "max_blocks": None, "x_len": 8000,
                  "y_len": 8000, "seed": 6001})
    out = []
    for c in cases:
        rng = np.random.default_rng(c["seed"])
        if c.get("zeros"):
            xb = yb = bytes(c["x_len"])
        else:
            xb, yb = rng.bytes(c["x_len"]), rng.bytes(c["y_len"])
        plan = R_params.plan_neq(c["b"], "3/4", c["q1"], c["growth"])
        sink = io.BytesIO()
        rep = R_ext.extract_neq(xb, yb, plan, max_blocks=c["max_blocks"]).run(sink)
        c = dict(c)
        c["out"] = sink.getvalue().hex()
        c["report"] = report_dict(rep)
        out.append(c)
    dump("neq_cases.json", out)


def make_pack():
    rng = np.random.default_rng(99)
    cases = []
    for b in range(1, 65):
        count = int(rng.integers(1, 90))
        hi = (1 << b) - 1
        vals = [int(v) & hi for v in rng.integers(0, 2**63, size=count, dtype=np.int64)]
        vals = [(v | (int(rng.integers(0, 2)) << 63)) & hi for v in vals]
        data = R_src._pack_samples(np.array(vals, dtype=np.uint64), b)
        cases.append({"b": b, "values": [h(v) for v in vals], "out": data.hex()})
    dump("pack.json", cases)


def make_c1():
    wl = W.WORKLOADS["c1"]
    xb = R_src.generate(R_src.iid_biased(0.5, seed=1), wl.samples)
    yb = R_src.generate(R_src.iid_biased(0.5, seed=2), wl.samples)
    plan = tiny_plan(1, wl.samples, 1, wl.n, wl.q)
    sink = io.BytesIO()
    rep = R_ext.extract_eq(xb, yb, plan).run(sink)
    out = sink.getvalue()
    (HERE / "c1_out.bin").write_bytes(out)
    dump("c1.json", {"x_sha256": hashlib.sha256(xb).hexdigest(),
                     "y_sha256": hashlib.sha256(yb).hexdigest(),
                     "out_sha256": hashlib.sha256(out).hexdigest(),
                     "report": report_dict(rep), "plan_log2_error": repr(plan.log2_error)})


def ref_generate(spec: W.SourceSpec, count: int) -> bytes:
    if spec.kind == "iid-biased":
        return R_src.generate(R_src.iid_biased(spec.p, seed=spec.seed), count)
    return R_src.generate(R_src.iid_table(list(spec.table), spec.bits_per_sample,
                                          seed=spec.seed), count)


def make_streams():
    out = {}
    for name in ("c1", "c2", "c3", "c5_n512", "paper"):
        wl = W.WORKLOADS[name]
        for side, spec in (("x", wl.x), ("y", wl.y)):
            count = 1 << 15
            ref = ref_generate(spec, count)
            mine = W.stream_bytes_host(spec, count, chunk=1 << 12).tobytes()
            assert ref == mine, (name, side)
            out[f"{name}.{side}"] = hashlib.sha256(ref).hexdigest()
    dump("streams.json", out)


def markov_table(b: int, table_seed: int) -> np.ndarray:
    """Transition table used by the markov fixtures (regenerated by the tests)."""
    size = 1 << b
    t = np.random.default_rng(table_seed).random((size, size)) ** 3
    return t / t.sum(axis=1, keepdims=True)


def make_markov():
    cases = []
    for b, count, seed in [(1, 5000, 3), (2, 4000, 4), (3, 3000, 5), (4, 3000, 6), (8, 2000, 7)]:
        t = markov_table(b, 31 + b)
        data = R_src.generate(R_src.markov(t, b, seed=seed), count)
        cases.append({"b": b, "count": count, "seed": seed, "table_seed": 31 + b, "out": data.hex()})
    dump("markov.json", cases)


def make_verify():
    from blockext import verify as R_v
    out = {"tables": {}, "bias": [], "distance": [], "hadamard": []}
    for q, n in [(1, 3), (2, 3), (3, 4), (4, 3), (5, 2), (6, 2), (12, 1), (2, 6)]:
        z = R_v.ip_value_table(R_gf.field(q), n)
        out["tables"][f"{q},{n}"] = hashlib.sha256(z.astype(np.uint16).tobytes()).hexdigest()
    for q, n, k, seed in [(2, 2, 2, 0), (2, 3, 3, 1), (3, 2, 4, 2), (4, 2, 5, 3), (1, 4, 2, 4)]:
        r = R_v.check_one_bit_bias(R_gf.field(q), n, k, seed=seed, sampled_pairs=60)
        out["bias"].append({"q": q, "n": n, "k": k, "seed": seed, "max_bias": repr(r.max_bias),
                            "bound": repr(r.bound), "pairs": r.pairs_tested,
                            "exhaustive": r.exhaustive})
    rng = np.random.default_rng(77)
    for q, n in [(2, 2), (3, 3), (4, 2), (2, 5)]:
        size = 1 << (q * n)
        px = rng.random(size) ** 4
        px /= px.sum()
        py = rng.random(size) ** 2
        py /= py.sum()
        r = R_v.check_extractor_distance(R_gf.field(q), n, px, py)
        out["distance"].append({"q": q, "n": n, "seed": 77, "distance": repr(r.distance),
                                "bound": repr(r.bound), "rate": repr(r.rate)})
    for q, n in [(1, 5), (2, 4), (3, 3), (5, 2), (9, 1), (4, 3)]:
        out["hadamard"].append({"q": q, "n": n,
                                "direct": R_v.check_hadamard(R_gf.field(q), n, method="direct")
                                if q * n <= 12 else None,
                                "counts": R_v.check_hadamard(R_gf.field(q), n, method="counts")})
    dump("verify.json", out)


def make_sampled():
    out = {}
    rnd = random.Random(4242)
    for name in ("c2", "c2p", "c3", "c5_n128", "c5_n256", "c5_n512", "c5_n1024",
                 "c5_n2048", "paper"):
        wl = W.WORKLOADS[name]
        nb = wl.num_blocks
        idx = sorted({0, 1, 2, nb // 2, nb - 1} | {rnd.randrange(nb) for _ in range(10)})
        B = wl.block_bits
        rows = []
        for l in idx:
            # window = stream bits [l*B, (l+1)*B); generate whole samples covering it
            b = wl.b
            s0 = (l * B) // b
            s1 = -(-((l + 1) * B) // b)
            # align to bytes for b=1 streams
            if b == 1:
                s0 -= s0 % 8
                s1 += (-s1) % 8
            xw = W.window_bytes(wl.x, s0 * b, (s1 - s0) * b)
            yw = W.window_bytes(wl.y, s0 * b, (s1 - s0) * b)
            skip = l * B - s0 * b
            xi = (int.from_bytes(xw, "little") >> skip) & ((1 << B) - 1)
            yi = (int.from_bytes(yw, "little") >> skip) & ((1 << B) - 1)
            ctx = R_gf.field(wl.q)
            xs = [(xi >> (j * wl.q)) & ctx.mask for j in range(wl.n)]
            ys = [(yi >> (j * wl.q)) & ctx.mask for j in range(wl.n)]
            z = R_ext.ext_ip(ctx, xs, ys)
            rows.append([l, h(z)])
        out[name] = {"q": wl.q, "n": wl.n, "blocks": rows}
    dump("sampled.json", out)


def main(argv):
    which = set(argv[1:]) or {"moduli", "gf", "ext_ip", "eq", "neq", "pack", "c1",
                              "streams", "sampled", "markov", "verify"}
    if "moduli" in which:
        make_moduli()
    if "gf" in which:
        make_gf()
    if "ext_ip" in which:
        make_ext_ip()
    if "eq" in which:
        make_eq_cases()
    if "neq" in which:
        make_neq_cases()
    if "pack" in which:
        make_pack()
    if "c1" in which:
        make_c1()
    if "streams" in which:
        make_streams()
    if "sampled" in which:
        make_sampled()
    if "markov" in which:
        make_markov()
    if "verify" in which:
        make_verify()
    print("reference blockext", blockext.__version__, file=sys.stderr)


if __name__ == "__main__":
    main(sys.argv)
