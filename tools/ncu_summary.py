#!/usr/bin/env python
"""Summarise an ncu --set full report (one kernel) into a short text block:
duration, DRAM bytes / throughput, tensor-pipe activity, issue utilisation and
the top stall reasons. Usage: python tools/ncu_summary.py report.ncu-rep [title]"""
import csv
import io
import subprocess
import sys


def raw(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return dict(zip(rows[0], rows[2])), dict(zip(rows[0], rows[1]))


SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1.0,
         "ms": 1e3, "Mhz": 1e6, "Ghz": 1e9, "hz": 1.0}


def num(d, k):
    try:
        return float(d[k].replace(",", ""))
    except Exception:
        return float("nan")


def main():
    path = sys.argv[1]
    title = sys.argv[2] if len(sys.argv) > 2 else path
    d, unit = raw(path)

    def val(k):
        return num(d, k) * SCALE.get(unit.get(k, ""), 1.0)

    dur_us = val("gpu__time_duration.sum")
    rd, wr = val("dram__bytes_read.sum"), val("dram__bytes_write.sum")
    lines = [f"== {title}", f"kernel: {d.get('Kernel Name', '?')}",
             f"duration: {dur_us:.1f} us",
             f"dram read: {rd / 1e6:.1f} MB  write: {wr / 1e6:.1f} MB  (traffic {rd + wr:.0f} B per launch)",
             f"achieved dram: {(rd + wr) / dur_us / 1e3:.0f} GB/s",
             f"dram throughput: {num(d, 'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed'):.1f}% of peak",
             f"tensor pipe active: {num(d, 'sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active'):.1f}% (of active cycles)",
             f"issue slots busy: {num(d, 'sm__inst_issued.avg.pct_of_peak_sustained_active'):.1f}%",
             f"warps active/SM: {num(d, 'sm__warps_active.avg.per_cycle_active'):.1f}",
             "top stall reasons (warps per issue):"]
    st = [(num(d, k), k.replace("smsp__average_warps_issue_stalled_", "").replace(
        "_per_issue_active.ratio", "")) for k in d if k.startswith("smsp__average_warps_issue_stalled_")
          and k.endswith("_per_issue_active.ratio")]
    for v, k in sorted(st, reverse=True)[:6]:
        lines.append(f"  {k:24s} {v:.2f}")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
