"""Render the per-workload bench lines under profiles/ as the markdown table in
profiles/r01_summary.md (python tools/bench_table.py [files...])."""
import glob
import json
import sys


def row(d):
    c, r, e = d["config"], d["roofline"], d.get("e2e") or {}
    cpu = d.get("cpu_baseline") or {}
    return "| {} | {} | {} | {:,.0f} | {:.1f} | {} | {:.3f} | {:,.0f} | {:.2f} | {} | {:.4f} |".format(
        c["workload"], c.get("q"), c.get("n"), d["value"], d.get("output_gbps", float("nan")),
        r["bound"], r["frac"], e.get("value") or 0.0, cpu.get("value") or float("nan"),
        (d.get("parity") or {}).get("mismatches"), d["ms_per_step"])


def main(paths):
    paths = paths or sorted(glob.glob("profiles/r01_bench_configs/*.json")) + ["profiles/r01_bench_c2_latest.json"]
    print("| workload | q | n | kernel raw Gbit/s | out Gbit/s | bound | frac | e2e raw Gbit/s "
          "| CPU port Gbit/s | sampled mismatches | ms/step |")
    print("|---|---|---|---|---|---|---|---|---|---|---|")
    for p in paths:
        print(row(json.load(open(p))))


if __name__ == "__main__":
    main(sys.argv[1:])
