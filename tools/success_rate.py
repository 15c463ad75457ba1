#!/usr/bin/env python3
"""Stochastic success-rate parity: the reference's IMS vs the B200 IMS on
BASELINE configs, over many seeds, to a FIXED target cut.

north_star: "Full stochastic runs must match the reference in success rate to
the best-known cut."  The paper reports medians over 30 runs
(PAPER.md:610-612); the reference's own statistical gate is
tests/test_engine_serial.cpp:237-262 (>= 29/30 seeds).

Per config a fixed target T (a cut the reference's IMS reaches in most runs,
chosen from its own pilot runs) and a fixed budget in gray-box evaluations E
(calls / q, the reference's RunControl::evaluations, runtime.hpp:95-99) —
machine-independent, so both sides get the same algorithmic budget — plus a
wall-clock safety limit.  Each seed runs
  CPU: oracle/_ref/ref_driver ims (run_parallel: IMS base 16, sub 4, the same
       FOS, every host thread), target T, budget E;
  GPU: run_gpu (the same IMS over GpuParallelEngine, Philox donors), target T,
       budget E;
and records success, evaluations to the target and seconds to the target
(both clocks from RunContext creation, model prebuilt).  Success rates are
compared with a two-proportion z-test and Fisher's exact test.

    python tools/success_rate.py --config c2 --seeds 30 --out profiles/r02/success_c2.json
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

REF = os.path.join(ROOT, "oracle", "_ref", "ref_driver")

# target cut, evaluation budget (gray-box units), wall safety limit (s)
STUDY = {
    "c1": dict(target=1110.0, evals=3000.0, wall=60.0),
    "c2": dict(target=103400.0, evals=22000.0, wall=120.0),
    "c3": dict(target=9600000.0, evals=450.0, wall=180.0),
}


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def reference_run(cfg, seed, target, evals, wall, workers):
    w = cfg["weights"]
    wspec = "unit" if w == "unit" else f"int:{w[1]}:{w[2]}"
    cmd = [REF, "ims", "--torus", str(cfg["width"]), str(cfg["height"]), "--weights", wspec, "--inst-seed", "1",
           "--fos", cfg["ref_fos"], "--seed", str(seed), "--ims", "--ims-base", "16", "--ims-sub", "4",
           "--workers", str(workers), "--target", repr(target), "--max-evals", repr(evals),
           "--max-seconds", repr(wall)]
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=wall * 3 + 600)
    if res.returncode != 0:
        raise RuntimeError(res.stderr)
    r = json.loads(res.stdout)
    hit = next(((t, e) for t, e, f in r["trace"] if f >= target), None)
    return {"reached": r["reason"] == "target-reached", "reason": r["reason"], "best": r["best"],
            "seconds_to_target": hit[0] if hit else None, "evaluations_to_target": hit[1] if hit else None,
            "evaluations": r["evaluations"], "populations": r["populations"], "run_seconds": r["seconds"]}


def gpu_run(P, seed, target, evals, wall):
    import paper_2203_08680_b200 as G

    sink = G.RecordingSink()
    r = G.run_gpu(P, G.TerminationConfig(target_fitness=target, max_evaluations=evals, max_seconds=wall),
                  seed=seed, use_ims=True, ims=G.ImsConfig(16, 4), sink=sink, mode="philox")
    hit = next((x for x in sink.rows if x.fitness >= target), None)
    return {"reached": r.reason == "target-reached", "reason": r.reason, "best": r.best_fitness,
            "seconds_to_target": hit.seconds if hit else None,
            "evaluations_to_target": hit.evaluations if hit else None, "evaluations": r.evaluations,
            "populations": r.populations, "run_seconds": r.seconds}


def quartiles(xs):
    xs = sorted(x for x in xs if x is not None)
    if not xs:
        return None
    if len(xs) == 1:
        return {"q1": xs[0], "median": xs[0], "q3": xs[0], "n": 1}
    q = statistics.quantiles(xs, n=4, method="inclusive")
    return {"q1": q[0], "median": q[1], "q3": q[2], "n": len(xs)}


def proportion_tests(k1, n1, k2, n2):
    from scipy import stats

    p = (k1 + k2) / (n1 + n2)
    se = (p * (1 - p) * (1 / n1 + 1 / n2)) ** 0.5
    z = ((k1 / n1) - (k2 / n2)) / se if se > 0 else 0.0
    return {"z": z, "p_two_sided_z": float(2 * stats.norm.sf(abs(z))),
            "p_fisher": float(stats.fisher_exact([[k1, n1 - k1], [k2, n2 - k2]])[1])}


def main():
    from bench import CONFIGS

    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2", choices=sorted(STUDY))
    ap.add_argument("--seeds", type=int, default=30)
    ap.add_argument("--first-seed", type=int, default=1)
    ap.add_argument("--workers", type=int, default=os.cpu_count() or 1)
    ap.add_argument("--out", default=None)
    ap.add_argument("--gpu-only", action="store_true")
    a = ap.parse_args()
    cfg, st = CONFIGS[a.config], STUDY[a.config]
    import paper_2203_08680_b200 as G
    from tools.time_to_target import warm_device

    warm_device()
    inst = G.generate_torus(cfg["width"], cfg["height"], cfg["weights"], 1)
    fos = G.univariate_fos(inst.num_vertices) if cfg["fos"] == "uni" else G.neighbourhood_fos(inst)
    G.GpuProblem(inst, fos)  # first-use loading, untimed
    t0 = time.perf_counter()
    P = G.GpuProblem(inst, fos)
    build_s = time.perf_counter() - t0
    rows = []
    for seed in range(a.first_seed, a.first_seed + a.seeds):
        row = {"seed": seed, "gpu": gpu_run(P, seed, st["target"], st["evals"], st["wall"])}
        if not a.gpu_only:
            row["cpu"] = reference_run(cfg, seed, st["target"], st["evals"], st["wall"], a.workers)
        rows.append(row)
        print(json.dumps(row), flush=True)
    out = {"config": cfg["workload"], "target_cut": st["target"], "evaluation_budget": st["evals"],
           "wall_limit_s": st["wall"], "seeds": [r["seed"] for r in rows], "ims": "base 16, subgenerations 4",
           "cpu": {"engine": f"reference run_parallel (ParallelEngine, {a.workers} threads)", "model": cpu_model(),
                   "threads": a.workers},
           "gpu": {"engine": "run_gpu (GpuParallelEngine, Philox donors)", "problem_build_s": build_s}}
    for side in ("gpu", "cpu"):
        if side not in rows[0]:
            continue
        rs = [r[side] for r in rows]
        k = sum(1 for x in rs if x["reached"])
        out[side].update({
            "success": k, "runs": len(rs), "success_rate": k / len(rs),
            "seconds_to_target": quartiles(x["seconds_to_target"] for x in rs),
            "evaluations_to_target": quartiles(x["evaluations_to_target"] for x in rs),
            "best_unreached": sorted(x["best"] for x in rs if not x["reached"])})
    if "cpu" in rows[0]:
        g, c = out["gpu"], out["cpu"]
        out["parity"] = proportion_tests(g["success"], g["runs"], c["success"], c["runs"])
        if g["seconds_to_target"] and c["seconds_to_target"]:
            out["speedup_median_seconds"] = c["seconds_to_target"]["median"] / g["seconds_to_target"]["median"]
            out["speedup_median_seconds_incl_build"] = \
                c["seconds_to_target"]["median"] / (g["seconds_to_target"]["median"] + build_s)
    out["rows"] = rows
    print(json.dumps({k: v for k, v in out.items() if k != "rows"}))
    if a.out:
        os.makedirs(os.path.dirname(os.path.abspath(a.out)), exist_ok=True)
        with open(a.out, "w") as fh:
            json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
