"""Stall-reason totals and the top stalled source lines of an ncu source page
(`ncu -i R --page source --csv --print-source cuda,sass > x.csv`)."""
import csv
import sys
from collections import defaultdict


def main(path, top=25):
    rows = list(csv.reader(open(path, errors="replace")))
    for i, r in enumerate(rows):
        if r and r[0] == "Line No":
            hdr, start = r, i + 1
            break
    st_cols = [j for j, h in enumerate(hdr) if h.startswith("stall_")]
    tot = defaultdict(int)
    per_line = defaultdict(lambda: defaultdict(int))
    src = {}
    line = None
    for r in rows[start:]:
        if len(r) < len(hdr):
            continue
        if r[0]:
            line = r[0]
            src[line] = r[1]
        for j in st_cols:
            try:
                v = int(r[j] or 0)
            except ValueError:
                continue
            tot[hdr[j]] += v
            per_line[line][hdr[j]] += v
    T = sum(tot.values()) or 1
    print("stall totals:", ", ".join(f"{k[6:]} {100 * v / T:.1f}%" for k, v in sorted(tot.items(), key=lambda kv: -kv[1]) if v))
    lines = sorted(per_line.items(), key=lambda kv: -sum(kv[1].values()))[:top]
    for ln, d in lines:
        s = sum(d.values())
        top3 = ", ".join(f"{k[6:]} {v}" for k, v in sorted(d.items(), key=lambda kv: -kv[1])[:3] if v)
        print(f"{100 * s / T:5.1f}%  L{ln:>5} [{top3}] {src.get(ln, '')[:90]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
