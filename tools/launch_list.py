#!/usr/bin/env python
"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list per kernel.

    python tools/launch_list.py launches.csv "title" "command" > profiles/rN_launches_X.csv
"""
import collections
import csv
import sys

SCALE = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}


def main():
    path, title, cmd = sys.argv[1], sys.argv[2], sys.argv[3]
    rows = list(csv.reader(open(path)))
    hdr = [r for r in rows if r and r[0] == "ID"][0]
    agg = collections.OrderedDict()
    for r in rows:
        if not r or r[0] == "ID" or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d["Metric Name"] != "gpu__time_duration.sum":
            continue
        us = float(d["Metric Value"].replace(",", "")) * SCALE[d["Metric Unit"]]
        a = agg.setdefault(d["Kernel Name"][:100], [0, 0.0])
        a[0] += 1
        a[1] += us
    tot = sum(a[1] for a in agg.values())
    print(f"# {title}: ncu --metrics gpu__time_duration.sum --clock-control none "
          "(cold-cache, serialised)")
    print(f"# command: {cmd}")
    print("kernel,launches,total_us,mean_us,share")
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"\"{k}\",{n},{t:.1f},{t / n:.2f},{t / tot:.3f}")


if __name__ == "__main__":
    main()
