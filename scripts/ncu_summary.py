"""Summarise .ncu-rep captures (--set full) into a small text table for profiles/."""
import csv, io, subprocess, sys

KEYS = ["Duration", "Elapsed Cycles", "SM Frequency", "DRAM Throughput", "Memory Throughput",
        "Compute (SM) Throughput", "L2 Hit Rate", "Registers Per Thread", "Dynamic Shared Memory Per Block",
        "Grid Size", "Block Size", "Achieved Occupancy"]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
       "sm__inst_executed_pipe_uniform.sum", "smsp__inst_executed.sum"]


def rows(rep, page, extra=()):
    out = subprocess.run(["ncu", "-i", rep, "--page", page, "--csv", *extra], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


for rep in sys.argv[1:]:
    print(f"== {rep}")
    r = rows(rep, "details")
    h = r[0]
    ki = h.index("Kernel Name")
    for row in r[1:]:
        if len(row) < len(h):
            continue
        if row[h.index("Metric Name")] in KEYS:
            print(f"  {row[ki][:40]:40s} {row[h.index('Metric Name')]:34s} {row[h.index('Metric Value')]:>12s} "
                  f"{row[h.index('Metric Unit')]}")
    r = rows(rep, "raw", ["--metrics", ",".join(RAW)])
    if len(r) > 2:
        h, units, vals = r[0], r[1], r[2]
        for m in RAW:
            if m in h:
                i = h.index(m)
                print(f"  raw {m:40s} {vals[i]:>16s} {units[i]}")
