"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list per kernel."""
import csv
import re
import sys
from collections import defaultdict


def short(name):
    name = re.sub(r"\(int\)|\(bool\)", "", name)
    name = name.replace("void ", "")
    base = name.split("(")[0]
    return base[:70]


def main(path):
    rows = list(csv.reader(open(path)))
    for i, r in enumerate(rows):
        if "Kernel Name" in r:
            hdr, start = r, i + 1
            break
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows[start:]:
        if len(r) <= vi:
            continue
        k = short(r[ki])
        agg[k][0] += 1
        agg[k][1] += float(r[vi].replace(",", ""))
    tot = sum(v[1] for v in agg.values())
    for k, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{k:70s} n={c:5d} total={t / 1e3:10.1f}us share={100 * t / tot:5.1f}% avg={t / c / 1e3:8.2f}us")


if __name__ == "__main__":
    main(sys.argv[1])
