#!/usr/bin/env python3
"""Per-source-line hot spots of an ncu report (--set full --import-source on, built with
-lineinfo): warp-stall samples and executed warp instructions per CUDA source line.

  ncu -i prof.ncu-rep --page source --csv --print-source cuda,sass > mix.csv
  python tools/ncu_lines.py mix.csv [top]
"""
import csv
import sys


def main(path, top=40):
    rows = list(csv.reader(open(path)))
    hdr = next(r for r in rows if r and r[0] == "Line No")
    i_st, i_ex = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
    lines = []
    for r in rows:
        if len(r) == len(hdr) and r[0] not in ("", "Line No"):
            try:
                lines.append((int(r[0]), r[1], float(r[i_st] or 0), float(r[i_ex] or 0)))
            except ValueError:
                pass
    tot_s = sum(x[2] for x in lines) or 1
    tot_e = sum(x[3] for x in lines) or 1
    print(f"total stall samples {tot_s:.0f}, warp instructions {tot_e:.3g}")
    for ln, src, st, ex in sorted(lines, key=lambda x: -x[2])[:top]:
        print(f"{ln:5d} {100 * st / tot_s:6.2f}% stalls {100 * ex / tot_e:6.2f}% inst  {src.strip()[:90]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
