"""Aggregate an `ncu --page source --csv --print-source cuda,sass` dump per CUDA
source line: executed instructions and warp-stall samples (top N)."""
import csv
import sys
from collections import defaultdict


def main(path, top=40):
    rows = list(csv.reader(open(path)))
    hdr = None
    for i, r in enumerate(rows):
        if r and r[0] == "Line No":
            hdr, start = r, i + 1
            break
    ex_i = hdr.index("Instructions Executed")
    st_i = hdr.index("Warp Stall Sampling (All Samples)")
    agg = defaultdict(lambda: [0, 0])
    src = {}
    line = None
    for r in rows[start:]:
        if len(r) <= ex_i:
            continue
        if r[0]:
            line = r[0]
            src[line] = r[1]
        try:
            agg[line][0] += int(r[ex_i] or 0)
            agg[line][1] += int(r[st_i] or 0)
        except ValueError:
            pass
    tot = sum(v[0] for v in agg.values())
    tst = sum(v[1] for v in agg.values())
    print(f"total instructions {tot}, stall samples {tst}")
    for ln, (ex, st) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f"{ex:10d} {100 * ex / tot:5.1f}%  stall {100 * st / max(tst, 1):5.1f}%  L{ln:>5} {src.get(ln, '')[:100]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
