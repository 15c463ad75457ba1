"""Aggregate an `ncu --page source --csv --print-source cuda,sass` dump per CUDA
source line (every file of the kernel): executed warp instructions and
warp-stall samples, top N."""
import csv
import os
import sys
from collections import defaultdict


def main(path, top=40):
    agg = defaultdict(lambda: [0, 0])
    src = {}
    hdr = None
    fname = "?"
    line = None
    for r in csv.reader(open(path)):
        if not r:
            continue
        if r[0] == "File Path":
            fname = os.path.basename(r[1])
            hdr = None
            continue
        if r[0] == "Line No":
            hdr = r
            ex_i = hdr.index("Instructions Executed")
            st_i = hdr.index("Warp Stall Sampling (All Samples)")
            continue
        if hdr is None or len(r) <= ex_i:
            continue
        if r[0]:
            line = (fname, r[0])
            src[line] = r[1]
        try:
            agg[line][0] += int(r[ex_i] or 0)
            agg[line][1] += int(r[st_i] or 0)
        except ValueError:
            pass
    tot = sum(v[0] for v in agg.values())
    tst = sum(v[1] for v in agg.values())
    print(f"total warp instructions {tot}, stall samples {tst}")
    for (f, ln), (ex, st) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f"{ex:10d} {100 * ex / tot:5.1f}%  stall {100 * st / max(tst, 1):5.1f}%  {f}:{ln:<5} "
              f"{src.get((f, ln), '').strip()[:90]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
