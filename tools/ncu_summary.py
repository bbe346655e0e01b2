"""Key metrics of an ncu --set full report (per kernel launch) for profiles/ summaries."""
import csv
import subprocess
import sys

WANT = ["Duration", "DRAM Throughput", "Memory Throughput", "L1/TEX Hit Rate", "L2 Hit Rate", "L1/TEX Cache Throughput",
        "L2 Cache Throughput", "Achieved Occupancy", "Theoretical Occupancy", "Registers Per Thread",
        "Dynamic Shared Memory Per Block", "Warp Cycles Per Issued Instruction", "Issue Slots Busy",
        "Compute (SM) Throughput", "Block Limit Registers", "Block Limit Shared Mem", "Grid Size", "Block Size"]


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    h = r[0]
    ki, mi, vi, ui, ii = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
    cur = None
    for row in r[1:]:
        if row[mi] not in WANT:
            continue
        if row[ii] != cur:
            cur = row[ii]
            print(f"== launch {cur}: {row[ki][:90]}")
        print(f"   {row[mi]:36s} {row[vi]:>14s} {row[ui]}")
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(raw.splitlines()))
    if len(rr) > 2:
        hh = rr[0]
        cols = [c for c in hh if c.startswith("dram__bytes_read.sum") or c.startswith("dram__bytes_write.sum")
                or c == "gpu__time_duration.sum" or c.startswith("smsp__average_warp") ]
        for row in rr[2:]:
            d = dict(zip(hh, row))
            print("   raw:", {c: d[c] for c in hh if c in ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum")},
                  "units:", {c: rr[1][hh.index(c)] for c in ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum") if c in hh})


if __name__ == "__main__":
    main(sys.argv[1])
