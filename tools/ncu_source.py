"""Per-(file, line) instructions and stall samples from an ncu source page
(`ncu -i R --page source --csv --print-source cuda,sass > x.csv`); the page
repeats a header block per source file and kernel.

    python tools/ncu_source.py x.csv [top] [--kernel SUBSTR]
"""
import csv
import os
import sys
from collections import defaultdict


def parse(path, kernel=None):
    rows = list(csv.reader(open(path, errors="replace")))
    agg = defaultdict(lambda: defaultdict(int))
    src = {}
    fname = func = None
    hdr = None
    line = None
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            fname = os.path.basename(r[1])
            continue
        if r[0] == "Function Name":
            func = r[1]
            continue
        if r[0] == "Line No":
            hdr = r
            cols = {h: j for j, h in enumerate(r)}
            continue
        if hdr is None or len(r) < len(hdr):
            continue
        if kernel and (func is None or kernel not in func):
            continue
        if r[0]:
            line = (fname, r[0])
            src[line] = r[1]
        d = agg[line]
        for h, j in cols.items():
            if h.startswith("stall_") or h == "Instructions Executed":
                try:
                    d[h] += int(r[j] or 0)
                except ValueError:
                    pass
    return agg, src


def main(path, top=30, kernel=None):
    agg, src = parse(path, kernel)
    tot_ins = sum(d["Instructions Executed"] for d in agg.values()) or 1
    stall_keys = {k for d in agg.values() for k in d if k.startswith("stall_") and "Not Issued" not in k}
    tot_st = sum(d[k] for d in agg.values() for k in stall_keys) or 1
    tot = defaultdict(int)
    for d in agg.values():
        for k in stall_keys:
            tot[k] += d[k]
    print("stall totals:", ", ".join(f"{k[6:]} {100 * v / tot_st:.1f}%" for k, v in
                                      sorted(tot.items(), key=lambda kv: -kv[1]) if v))
    print(f"{'stall%':>6} {'inst%':>6}  file:line")
    key = lambda kv: -sum(kv[1][k] for k in stall_keys)
    for ln, d in sorted(agg.items(), key=key)[:top]:
        st = sum(d[k] for k in stall_keys)
        top3 = ", ".join(f"{k[6:]} {d[k]}" for k in sorted(stall_keys, key=lambda k: -d[k])[:2] if d[k])
        print(f"{100 * st / tot_st:6.1f} {100 * d['Instructions Executed'] / tot_ins:6.1f}  "
              f"{ln[0]}:{ln[1]} [{top3}] {src.get(ln, '')[:80]}")


if __name__ == "__main__":
    args = [a for a in sys.argv[1:] if not a.startswith("--kernel")]
    kern = next((a.split("=", 1)[1] for a in sys.argv[1:] if a.startswith("--kernel=")), None)
    main(args[0], int(args[1]) if len(args) > 1 else 30, kern)
