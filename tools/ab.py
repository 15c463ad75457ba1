#!/usr/bin/env python3
"""A/B timing of library builds / environment switches on one box, runs
interleaved so clocks and box-to-box variation cancel:

    python tools/ab.py [--config c3] [--rounds 5] [--gens 200] \
        base "rot:GOMIX_LIB=paper_2203_08680_b200/libgomix_b200_rot.so" "direct:GOMIX_GRAPH=0"

Each spec is NAME[:VAR=VALUE[,VAR=VALUE...]]; every (round, spec) runs in a
fresh process: the CONFIG's problem, a Philox engine, `gens` queued
generations after warm-up, CUDA events around them.  Prints the median
ms/generation and throughput per spec."""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import json, sys, os
sys.path.insert(0, {root!r}); sys.path.insert(0, os.path.join({root!r}, "tools"))
import paper_2203_08680_b200 as G
from bench import CONFIGS
from sweep import device_rate
if {config!r}.startswith("c4"):  # c4 / c4d16: random d-regular, 1e5 vertices, fp64 weights, univariate, n = 128
    deg = int({config!r}[3:]) if len({config!r}) > 2 else 4
    n = {n} or 128
    inst = G.generate_regular(100000, deg, ("real",), seed=deg)
    fos = G.univariate_fos(inst.num_vertices)
else:
    cfg = CONFIGS[{config!r}]
    n = {n} or cfg["n"]
    inst = G.generate_torus(cfg["width"], cfg["height"], cfg["weights"], 1)
    fos = G.univariate_fos(inst.num_vertices) if cfg["fos"] == "uni" else G.neighbourhood_fos(inst)
P = G.GpuProblem(inst, fos)
r = device_rate(G, P, n, gens={gens}, warm=10, flush={flush})
print("RESULT " + json.dumps(r))
"""


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("specs", nargs="+")
    ap.add_argument("--config", default="c3")
    ap.add_argument("--n", type=int, default=0)
    ap.add_argument("--rounds", type=int, default=5)
    ap.add_argument("--gens", type=int, default=200)
    ap.add_argument("--flush", action="store_true", help="flush L2 between generations (the bench's condition)")
    args = ap.parse_args()
    specs = []
    for s in args.specs:
        name, _, envs = s.partition(":")
        env = dict(e.split("=", 1) for e in envs.split(",") if e)
        specs.append((name, env))
    code = CHILD.format(root=ROOT, config=args.config, n=args.n, gens=args.gens, flush=args.flush)
    res = {name: [] for name, _ in specs}
    for rnd in range(args.rounds):
        for name, env in specs:
            e = dict(os.environ)
            e.update(env)
            out = subprocess.run([sys.executable, "-c", code], env=e, cwd=ROOT, capture_output=True, text=True,
                                 timeout=600)
            line = [l for l in out.stdout.splitlines() if l.startswith("RESULT ")]
            if not line:
                print(f"{name}: failed\n{out.stderr[-2000:]}", flush=True)
                continue
            r = json.loads(line[0][7:])
            res[name].append(r)
            print(f"round {rnd} {name}: {r['ms_per_generation'] * 1e3:.2f} us/gen {r['steps_per_s']:.4g}/s",
                  flush=True)
    summary = {}
    for name, rs in res.items():
        if rs:
            summary[name] = {"median_us_per_gen": round(statistics.median(r["ms_per_generation"] for r in rs) * 1e3, 3),
                             "median_steps_per_s": statistics.median(r["steps_per_s"] for r in rs),
                             "kernel": rs[0]["kernel"], "runs": len(rs)}
    print(json.dumps({"config": args.config, "gens": args.gens, "summary": summary}, indent=1))


if __name__ == "__main__":
    main()
