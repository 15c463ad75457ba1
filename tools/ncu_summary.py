"""Key metrics of every kernel in an .ncu-rep (`ncu -i … --page details --csv`)."""
import csv
import io
import subprocess
import sys

KEYS = ["Duration", "Elapsed Cycles", "SM Active Cycles", "DRAM Throughput", "Memory Throughput",
        "L2 Cache Throughput", "L1/TEX Cache Throughput", "Compute (SM) Throughput", "Executed Ipc Active",
        "Issue Slots Busy", "Registers Per Thread", "Achieved Active Warps Per SM", "Theoretical Occupancy",
        "Achieved Occupancy", "Executed Instructions", "Warp Cycles Per Issued Instruction", "L2 Hit Rate",
        "L1/TEX Hit Rate", "Grid Size", "Block Size", "Static Shared Memory Per Block",
        "Dynamic Shared Memory Per Block", "Avg. Active Threads Per Warp"]


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[0]
    ki, mi, vi, ui, ii = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
    seen = {}
    for r in rows[1:]:
        if len(r) <= vi or r[mi] not in KEYS:
            continue
        seen.setdefault((r[ii], r[ki][:90]), {})[r[mi]] = f"{r[vi]} {r[ui]}".strip()
    for (i, k), d in seen.items():
        print(f"[{i}] {k}")
        for key in KEYS:
            if key in d:
                print(f"    {key:40s} {d[key]}")
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    hdr = rr[0]
    want = [c for c in hdr if c in ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum")]
    for r in rr[2:]:
        print("raw:", {c: r[hdr.index(c)] for c in want}, "units:", {c: rr[1][hdr.index(c)] for c in want})


if __name__ == "__main__":
    main(sys.argv[1])
