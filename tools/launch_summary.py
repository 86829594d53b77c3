# SPDX-License-Identifier: Apache-2.0
"""Summarise an ncu --csv launch list (gpu__time_duration.sum) by kernel:
launches, total time, share. Usage: python tools/launch_summary.py file.csv"""
import collections
import csv
import sys


def main(path):
    rows = list(csv.reader(open(path)))
    hdr, agg = None, collections.defaultdict(lambda: [0, 0.0])
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6, "s": 1e6}[d["Metric Unit"]]
        v = float(d["Metric Value"].replace(",", "")) * scale
        k = d["Kernel Name"].split("(")[0][:70]
        agg[k][0] += 1
        agg[k][1] += v
    tot = sum(v[1] for v in agg.values())
    print(f"{'launches':>8} {'total us':>12} {'avg us':>10} {'share':>6}  kernel")
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{n:8d} {t:12.1f} {t / n:10.1f} {100 * t / tot:5.1f}%  {k}")


if __name__ == "__main__":
    main(sys.argv[1])
