"""Summarise .ncu-rep captures into profiles/ (JSON + markdown table).

    python tools/ncu_summary.py gpurun_out/prof_c2b.ncu-rep:c2 ... --out profiles/r01_ncu
"""
import argparse
import csv
import io
import json
import subprocess
import sys

METRICS = [
    ("kernel", "Kernel Name"),
    ("duration_us", "gpu__time_duration.sum"),
    ("dram_read_bytes", "dram__bytes_read.sum"),
    ("dram_write_bytes", "dram__bytes_write.sum"),
    ("dram_pct_peak", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
    ("sm_throughput_pct", "sm__throughput.avg.pct_of_peak_sustained_elapsed"),
    ("alu_pipe_pct", "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active"),
    ("fma_pipe_pct", "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active"),
    ("lsu_pipe_pct", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active"),
    ("warps_active_pct", "sm__warps_active.avg.pct_of_peak_sustained_active"),
    ("l1tex_pct", "l1tex__throughput.avg.pct_of_peak_sustained_active"),
    ("issue_pct", "sm__inst_issued.avg.pct_of_peak_sustained_active"),
    ("registers", "launch__registers_per_thread"),
    ("grid", "launch__grid_size"),
    ("block", "launch__block_size"),
    ("inst_executed", "smsp__inst_executed.sum"),
    ("sm_clock_hz", "sm__cycles_elapsed.avg.per_second"),
]
SCALE = {"Mbyte": 1e6, "Gbyte": 1e9, "Kbyte": 1e3, "byte": 1, "usecond": 1, "msecond": 1e3, "ms": 1e3, "us": 1, "ns": 1e-3,
         "nsecond": 1e-3, "Ghz": 1e9, "Mhz": 1e6, "hz": 1}


def summarise(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, out = rows[0], rows[1], []
    for vals in rows[2:]:
        d = {}
        for key, name in METRICS:
            if name not in hdr:
                continue
            i = hdr.index(name)
            v = vals[i]
            try:
                f = float(v.replace(",", ""))
                f *= SCALE.get(units[i], 1)
                d[key] = f
            except ValueError:
                d[key] = v
        out.append(d)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("reps", nargs="+", help="file.ncu-rep:label")
    ap.add_argument("--out", required=True)
    a = ap.parse_args()
    res = {}
    for spec in a.reps:
        path, label = spec.rsplit(":", 1)
        res[label] = summarise(path)
    with open(a.out + ".json", "w") as f:
        json.dump(res, f, indent=1)
    lines = ["| workload | kernel | us | DRAM R+W MB | DRAM % | ALU % | FMA % | LSU % | L1 % | issue % | warps % | regs |",
             "|---|---|---|---|---|---|---|---|---|---|---|---|"]
    for label, ks in res.items():
        for k in ks:
            mb = (k.get("dram_read_bytes", 0) + k.get("dram_write_bytes", 0)) / 1e6
            lines.append(f"| {label} | {str(k.get('kernel'))[:40]} | {k.get('duration_us', 0):.1f} | {mb:.1f} | "
                         f"{k.get('dram_pct_peak', 0):.1f} | {k.get('alu_pipe_pct', 0):.1f} | "
                         f"{k.get('fma_pipe_pct', 0):.1f} | {k.get('lsu_pipe_pct', 0):.1f} | "
                         f"{k.get('l1tex_pct', 0):.1f} | {k.get('issue_pct', 0):.1f} | "
                         f"{k.get('warps_active_pct', 0):.1f} | {k.get('registers', 0):.0f} |")
    with open(a.out + ".md", "w") as f:
        f.write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    sys.exit(main())
