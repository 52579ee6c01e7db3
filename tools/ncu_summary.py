#!/usr/bin/env python3
"""Key metrics per kernel from an ncu raw page (ncu -i rep --page raw --csv > raw.csv), for the
profiles/ summaries: duration, DRAM bytes and throughput, pipe utilisation, occupancy.

  python tools/ncu_summary.py gpurun_out/r2_tc_adam.raw.csv [algorithmic_bytes_per_launch]
"""
import csv
import sys

METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
           "launch__grid_size", "launch__block_size", "sm__warps_active.avg.pct_of_peak_sustained_active",
           "smsp__inst_executed.sum", "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
           "lts__t_sectors_srcunit_tex_op_read.sum", "sm__cycles_elapsed.avg.per_second"]


def main(path, alg=None):
    rows = list(csv.reader(open(path)))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        if len(r) != len(hdr):
            continue
        print(f"Kernel Name  {r[hdr.index('Kernel Name')]}")
        vals = {}
        for m in METRICS:
            if m in hdr:
                i = hdr.index(m)
                vals[m] = (r[i], units[i])
                print(f"  {m:70s} {r[i]:>20s} {units[i]}")
        if alg and "dram__bytes_read.sum" in vals:
            def to_b(v, u):
                f = float(v.replace(",", ""))
                return f * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(u, 1)
            tot = to_b(*vals["dram__bytes_read.sum"]) + to_b(*vals["dram__bytes_write.sum"])
            print(f"  dram read+write {tot / 1e9:.3f} GB against {alg / 1e9:.3f} GB algorithmic ({tot / alg:.3f}x)")
            alg = None  # the first kernel only


if __name__ == "__main__":
    main(sys.argv[1], float(sys.argv[2]) if len(sys.argv) > 2 else None)
