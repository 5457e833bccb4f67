"""Command-line front end for the data-path subcommands.

    python -m paper_2402_14607_b200 params      --b 16 --delta 10.74/16 --N 2^47 --epsilon 2^-30
    python -m paper_2402_14607_b200 extract-eq  --x X --y Y --out OUT --b 8 --delta 3/4 --epsilon 2^-30
    python -m paper_2402_14607_b200 extract-neq --x X --y Y --out OUT --b 8 --delta 3/4 --q1 8

Same flags, output files, report text and exit codes as the reference CLI's
``params`` / ``extract-eq`` / ``extract-neq`` (pkg/src/blockext/cli.py:44-140,
333-427): 0 ok, 2 usage, 3 capacity, 4 unsupported rate, 5 I/O.  Extraction
runs on the GPU; file inputs stream through the bulk BitReader replay and the
pipelined host->device path.  The reference's simulate/verify/bench
subcommands are analytics outside the data path and are not provided.
"""
from __future__ import annotations

import argparse
import os
import sys

from .errors import CapacityError, TruncatedSourceError, UnsupportedRateError
from .extractor import extract_eq, extract_neq
from .params import as_rational, parse_count, parse_probability, plan_eq, plan_neq
from .report import plan_to_text

EXIT_USAGE, EXIT_CAPACITY, EXIT_RATE, EXIT_IO = 2, 3, 4, 5


def _plan_flags(p: argparse.ArgumentParser, need_n: bool = True) -> None:
    p.add_argument("--b", required=True, help="bits per sample, e.g. 16")
    p.add_argument("--delta", required=True, help="min-entropy rate, e.g. 10.74/16")
    p.add_argument("--epsilon", required=True, help="target distance, e.g. 2^-30")
    g = p.add_mutually_exclusive_group(required=need_n)
    g.add_argument("--N", help="samples per source, e.g. 2^47")
    g.add_argument("--N-bits", dest="n_bits", help="raw bits per source; must divide by --b")


def _eq_plan(args, default_samples: int | None = None):
    b = int(args.b)
    if args.N is not None:
        samples = parse_count(args.N)
    elif args.n_bits is not None:
        bits = parse_count(args.n_bits)
        if bits % b:
            raise ValueError(f"--N-bits {bits} is not a multiple of --b {b}")
        samples = bits // b
    elif default_samples is not None:
        samples = default_samples
    else:
        raise ValueError("need --N or --N-bits")
    return plan_eq(b, samples, as_rational(args.delta, "delta"), parse_probability(args.epsilon))


def _emit(text: str, path: str | None) -> None:
    if path:
        with open(path, "w") as fh:
            fh.write(text)
    else:
        sys.stdout.write(text)


class _Pair:
    """The two input streams; at most one may be standard input."""

    def __init__(self, x: str, y: str):
        if x == "-" and y == "-":
            raise ValueError("the two sources must be physically independent streams; "
                             "at most one may be standard input")
        self._paths = (x, y)
        self._fh = []

    def __enter__(self):
        for p in self._paths:
            self._fh.append(sys.stdin.buffer if p == "-" else open(p, "rb"))
        return self._fh

    def __exit__(self, *exc):
        for p, fh in zip(self._paths, self._fh):
            if p != "-":
                fh.close()
        return False


def _devices(args) -> dict:
    """--devices 0,1,2: shard every segment's blocks across these GPUs."""
    if not getattr(args, "devices", None):
        return {}
    return {"devices": [f"cuda:{int(d)}" for d in args.devices.split(",") if d.strip()]}


def cmd_params(args) -> int:
    _emit(plan_to_text(_eq_plan(args)), args.report)
    return 0


def cmd_extract_eq(args) -> int:
    default = None
    if args.N is None and args.n_bits is None:
        if "-" in (args.x, args.y):
            raise ValueError("--N or --N-bits is required when reading standard input")
        usable = min(os.path.getsize(args.x), os.path.getsize(args.y))
        default = usable * 8 // int(args.b)
    plan = _eq_plan(args, default)
    with _Pair(args.x, args.y) as (fx, fy), open(args.out, "wb") as out:
        report = extract_eq(fx, fy, plan, workers=args.workers, **_devices(args)).run(out)
    _emit(report.to_text(), args.report)
    return 0


def cmd_extract_neq(args) -> int:
    plan = plan_neq(int(args.b), as_rational(args.delta, "delta"),
                    first_field_bits=int(args.q1), growth=int(args.growth))
    with _Pair(args.x, args.y) as (fx, fy), open(args.out, "wb") as out:
        report = extract_neq(fx, fy, plan, workers=args.workers,
                             max_blocks=args.max_blocks).run(out)
    _emit(report.to_text(), args.report)
    return 0


def build_parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="blockext-b200",
                                 description="B200 two-source extraction for block sources")
    sub = ap.add_subparsers(dest="command", required=True)
    p = sub.add_parser("params", help="derive and print an equal-block plan")
    _plan_flags(p)
    p.add_argument("--report")
    p.set_defaults(func=cmd_params)
    p = sub.add_parser("extract-eq", help="equal-block extraction of two files")
    p.add_argument("--x", required=True)
    p.add_argument("--y", required=True)
    p.add_argument("--out", required=True)
    _plan_flags(p, need_n=False)
    p.add_argument("--workers", type=int, default=1)
    p.add_argument("--devices", help="comma-separated CUDA device indices to shard across")
    p.add_argument("--report")
    p.set_defaults(func=cmd_extract_eq)
    p = sub.add_parser("extract-neq", help="incremental-block extraction")
    for f in ("--x", "--y", "--out", "--b", "--delta", "--q1"):
        p.add_argument(f, required=True)
    p.add_argument("--growth", default=1)
    p.add_argument("--max-blocks", type=int, default=None)
    p.add_argument("--workers", type=int, default=1)
    p.add_argument("--report")
    p.set_defaults(func=cmd_extract_neq)
    return ap


def main(argv=None) -> int:
    args = build_parser().parse_args(argv)
    try:
        return args.func(args)
    except UnsupportedRateError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return EXIT_RATE
    except CapacityError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return EXIT_CAPACITY
    except (OSError, TruncatedSourceError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return EXIT_IO
    except (ValueError, TypeError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return EXIT_USAGE


if __name__ == "__main__":
    sys.exit(main())
