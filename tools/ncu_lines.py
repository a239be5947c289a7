#!/usr/bin/env python
"""Top source lines by warp-stall samples from an ncu report (needs -lineinfo and
--import-source on). Usage: python tools/ncu_lines.py report.ncu-rep [N]"""
import csv
import io
import subprocess
import sys


def main():
    path = __import__("os").path.abspath(sys.argv[1])
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source=cuda,sass"],
                         capture_output=True, text=True, cwd="/tmp").stdout
    rows, cur, hdr = [], None, None
    for rec in csv.reader(io.StringIO(out)):
        if not rec:
            continue
        if rec[0] == "File Path":
            cur = rec[1].split("/")[-1]
            continue
        if rec[0] == "Line No":
            hdr = rec
            continue
        if hdr is None or not rec[0].isdigit() or rec[2] != "-":
            continue  # only the per-source-line aggregate rows
        d = dict(zip(hdr[:2], rec[:2]))
        vals = rec[4:]
        names = hdr[4:]
        m = {k: v for k, v in zip(names, vals)}
        try:
            samples = int(m.get("Warp Stall Sampling (All Samples)", "0").replace(",", ""))
        except ValueError:
            continue
        stalls = {k: int(v.replace(",", "")) for k, v in m.items()
                  if k.startswith("stall_") and "Not Issued" not in k and v.replace(",", "").isdigit()}
        top = sorted(stalls.items(), key=lambda kv: -kv[1])[:3]
        rows.append((samples, f"{cur}:{d['Line No']}", d["Source"].strip()[:70], top))
    tot = sum(r[0] for r in rows)
    print(f"total samples {tot}")
    for s, loc, src, top in sorted(rows, key=lambda r: -r[0])[:n]:
        print(f"{s:8d} {100 * s / tot:5.1f}%  {loc:22s} {src:70s} {' '.join(f'{k[6:]}={v}' for k, v in top)}")


if __name__ == "__main__":
    main()
