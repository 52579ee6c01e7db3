#!/usr/bin/env python3
"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv): launches, mean and
total time per kernel, and each kernel's share of the library's (dmb::) time."""
import collections
import csv
import sys


def main(path):
    hdr = None
    agg = collections.defaultdict(lambda: [0, 0.0])
    scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6, "s": 1e6}
    with open(path) as f:
        for r in csv.reader(f):
            if len(r) > 5 and r[0] == "ID":
                hdr = r
                continue
            if not hdr or len(r) != len(hdr):
                continue
            d = dict(zip(hdr, r))
            if d.get("Metric Name") != "gpu__time_duration.sum":
                continue
            us = float(d["Metric Value"].replace(",", "")) * scale.get(d["Metric Unit"], 1.0)
            name = d["Kernel Name"]
            agg[name][0] += 1
            agg[name][1] += us
    dmb = sum(t for n, (c, t) in agg.items() if "dmb::" in n)
    print(f"{'kernel':90s} {'launches':>8s} {'mean us':>10s} {'total us':>11s} {'dmb share':>9s}")
    for n, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        share = f"{100 * t / dmb:8.1f}%" if "dmb::" in n and dmb else "   (setup)"
        print(f"{n[:90]:90s} {c:8d} {t / c:10.1f} {t:11.1f} {share}")


if __name__ == "__main__":
    main(sys.argv[1])
