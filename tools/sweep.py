#!/usr/bin/env python3
"""BASELINE configs C4 and C5 as sweeps.

C4: random d-regular graphs, 10^5 vertices, fp64 weights uniform [0,1),
    univariate FOS, n = 128: colour-class count k per d and device throughput.
C5: 316x316 torus (~10^5 vertices), integer weights U[1,10], univariate FOS,
    population n = 16..4096: device throughput per n, and the reference
    ParallelEngine's throughput on the host cores at a few n (bounded sample).

Throughput = partial evaluations (executed (solution, set) pairs) per second,
CUDA events around G Philox generations after W warm-up generations.

    python tools/sweep.py [--c4] [--c5] [--out-dir profiles/r01]
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def hbm_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"])
    except (OSError, KeyError, ValueError):
        return 6650.0


def device_rate(G, P, n, gens=20, warm=3, seed=1, flush=False, **kw):
    """Queued Philox generations timed with CUDA events on the engine stream.
    flush: write 256 MiB between generations (outside the events), the
    bench's L2 condition."""
    import torch

    s = torch.cuda.Stream()
    E = G.GpuParallelEngine(P, n, seed, mode="philox", stream=s.cuda_stream, **kw)
    for _ in range(warm):
        E.run_generation_async()
    E.synchronize()
    _, st0, _ = E.group_counters()
    if flush:
        buf = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(gens)]
        with torch.cuda.stream(s):
            for a, b in ev:
                buf.fill_(1)
                a.record(s)
                E.run_generation_async()
                b.record(s)
        E.synchronize()
        torch.cuda.synchronize()
        ms = sum(a.elapsed_time(b) for a, b in ev)
    else:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(gens):
            E.run_generation_async()
        e1.record(s)
        E.synchronize()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
    _, st1, _ = E.group_counters()
    steps = int((st1 - st0).sum())
    return {"population": n, "steps_per_s": steps / (ms / 1e3), "ms_per_generation": ms / gens,
            "kernel": E.kernel_name(), "elitist": E.elitist_fitness}


def c4(G):
    rows = []
    for d in (4, 6, 8, 12, 16):
        inst = G.generate_regular(100000, d, ("real",), seed=d)
        t0 = time.perf_counter()
        P = G.GpuProblem(inst, G.univariate_fos(inst.num_vertices))
        build = time.perf_counter() - t0
        r = device_rate(G, P, 128)
        r.update({"degree": d, "colour_classes": P.num_groups, "bound_d_plus_1": d + 1,
                  "group_sizes": [len(g) for g in P.groups], "build_s": build, "exact": P.exact})
        rows.append(r)
        print(json.dumps({k: v for k, v in r.items() if k != "group_sizes"}), flush=True)
    return {"config": "C4: random d-regular, 1e5 vertices, fp64 weights U[0,1), univariate FOS, n=128",
            "rows": rows}


def c5(G, ref_points=(16, 64, 256)):
    from bench import CONFIGS, run_reference

    inst = G.generate_torus(316, 316, ("int", 1, 10), 1)
    P = G.GpuProblem(inst, G.univariate_fos(inst.num_vertices))
    rows = []
    peak = hbm_peak()
    for n in (16, 32, 64, 128, 256, 512, 1024, 2048, 4096):
        r = device_rate(G, P, n, gens=20 if n <= 1024 else 8)
        # B_step = 0.875 + 60 / n bytes for a degree-4 torus vertex
        r["bytes_per_step"] = 0.875 + 60.0 / n
        r["hbm_frac"] = r["steps_per_s"] * r["bytes_per_step"] / 1e9 / peak
        if n > 128:
            r["adder_kernel_steps_per_s"] = device_rate(G, P, n, gens=8, truth_table=False)["steps_per_s"]
        rows.append(r)
        print(json.dumps(r), flush=True)
    cfg = dict(CONFIGS["c5"])
    ref = []
    workers = os.cpu_count() or 1
    if ref_points and os.path.exists(os.path.join(ROOT, "oracle", "_ref", "ref_driver")):
        for n in ref_points:
            out = run_reference(cfg, n, 2, workers, timeout=900)
            secs = sum(g["seconds"] for g in out["gens"])
            st = sum(g["steps"] for g in out["gens"])
            ref.append({"population": n, "steps_per_s": st / secs, "workers": workers})
            print(json.dumps(ref[-1]), flush=True)
    return {"config": "C5: torus 316x316, integer weights U[1,10], univariate FOS, n = 16..4096",
            "rows": rows, "reference_cpu": ref}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--c4", action="store_true")
    ap.add_argument("--c5", action="store_true")
    ap.add_argument("--out-dir", default="gpurun_out")
    ap.add_argument("--no-ref", action="store_true", help="skip the reference CPU points")
    a = ap.parse_args()
    import paper_2203_08680_b200 as G

    os.makedirs(a.out_dir, exist_ok=True)
    if a.c4 or not (a.c4 or a.c5):
        json.dump(c4(G), open(os.path.join(a.out_dir, "sweep_c4.json"), "w"), indent=1)
    if a.c5 or not (a.c4 or a.c5):
        json.dump(c5(G, () if a.no_ref else (16, 64, 256)), open(os.path.join(a.out_dir, "sweep_c5.json"), "w"),
                  indent=1)


if __name__ == "__main__":
    main()
