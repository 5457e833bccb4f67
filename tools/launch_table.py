"""Markdown summary of an `ncu --metrics gpu__time_duration.sum --csv` launch list.

    python tools/launch_table.py gpurun_out/launches.csv "command" > profiles/rNN_launches_X.md
"""
import collections
import csv
import sys


def main(path, cmd):
    rows = []
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    for r in csv.DictReader(lines):
        if r.get("Metric Name") == "gpu__time_duration.sum":
            scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(r["Metric Unit"], 1e-3)
            rows.append((r["Kernel Name"], float(r["Metric Value"].replace(",", "")) * scale))
    agg = collections.OrderedDict()
    for name, us in rows:
        n, t = agg.get(name, (0, 0.0))
        agg[name] = (n + 1, t + us)
    total = sum(t for _, t in agg.values())
    print(f"ncu --metrics gpu__time_duration.sum --clock-control none of `{cmd}` "
          "(cold-cache, serialised; input generation and e2e legs included)\n")
    print("| kernel | launches | total us | mean us | share |")
    print("|---|---|---|---|---|")
    for name, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"| {name[:70]} | {n} | {t:.1f} | {t / n:.1f} | {100 * t / total:.1f}% |")
    seq = [(name, us) for name, us in rows if "bx::eq_" in name]
    if seq:
        print("\nExtraction launches in order (us): " + ", ".join(f"{us:.1f}" for _, us in seq))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "")
