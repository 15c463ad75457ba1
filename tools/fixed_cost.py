#!/usr/bin/env python3
"""Fixed cost per generation of the univariate path: ms/generation of the
C3 workload shape (torus, integer weights U[1,10], univariate FOS, Philox,
CUDA-graph generations) over torus sizes, and the straight-line fit
ms = fixed + per_pair * pairs.

    python tools/fixed_cost.py [--n 128] [--out profiles/r02/fixed_cost.json]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=128)
    ap.add_argument("--sides", default="8,16,32,64,100,200,316,500,707,1000")
    ap.add_argument("--gens", type=int, default=50)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    import numpy as np

    import paper_2203_08680_b200 as G
    from sweep import device_rate

    rows = []
    for side in (int(s) for s in args.sides.split(",")):
        inst = G.generate_torus(side, side, ("int", 1, 10), 1)
        P = G.GpuProblem(inst, G.univariate_fos(inst.num_vertices))
        r = device_rate(G, P, args.n, gens=args.gens, warm=10)
        r.update({"side": side, "vertices": side * side, "groups": P.num_groups,
                  "pairs_per_generation": side * side * args.n})
        rows.append(r)
        print(json.dumps(r), flush=True)
    big = [r for r in rows if r["vertices"] >= 10000]
    x = np.array([r["pairs_per_generation"] for r in big], dtype=np.float64)
    y = np.array([r["ms_per_generation"] for r in big])
    slope, icept = np.polyfit(x, y, 1)
    fit = {"fixed_ms_per_generation": float(icept), "ns_per_1e3_pairs": float(slope * 1e9),
           "fit_over": "sides with >= 1e4 vertices"}
    print(json.dumps(fit))
    if args.out:
        with open(args.out, "w") as fh:
            json.dump({"config": f"torus, int weights U[1,10], univariate FOS, n={args.n}, Philox, graph path",
                       "rows": rows, "fit": fit}, fh, indent=1)


if __name__ == "__main__":
    main()
