"""Headline metrics per launch from an ncu details page
(`ncu -i R --page details --csv > x.csv`).

    python tools/ncu_details.py x.csv
"""
import csv
import sys

WANT = ["Duration", "Executed Ipc Active", "Issue Slots Busy", "Registers Per Thread", "Theoretical Occupancy",
        "Achieved Occupancy", "Executed Instructions", "DRAM Throughput", "Memory Throughput", "L1/TEX Hit Rate",
        "L2 Hit Rate", "Warp Cycles Per Issued Instruction", "Grid Size", "Block Size",
        "Dynamic Shared Memory Per Block", "Static Shared Memory Per Block"]


def main(path):
    rows = list(csv.reader(open(path, errors="replace")))
    h = rows[0]
    ii, ki, mi, vi, ui = (h.index(x) for x in ("ID", "Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
    last = None
    for r in rows[1:]:
        if len(r) <= max(ii, ki, mi, vi, ui) or r[mi] not in WANT:
            continue
        if r[ii] != last:
            print(f"[{r[ii]}] {r[ki][:90]}")
            last = r[ii]
        print(f"    {r[mi]:<40} {r[vi]} {r[ui]}")


if __name__ == "__main__":
    main(sys.argv[1])
