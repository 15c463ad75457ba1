#!/usr/bin/env python3
"""Benchmark of the B200 GOM engine on BASELINE.json's headline metric.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c2]

One step = one GOM generation (ParallelEngine::run_generation,
engine_parallel.hpp:283-316) of the workload; the unit of work is one partial
evaluation = one executed (solution, linkage set) GOM step
(RunResult::GroupCounter::steps, runtime.hpp:170-175).

Default workload: BASELINE.json configs[2] = C3, Max-Cut 2-D torus 1000x1000
(10^6 vertices), integer weights U[1,10] (generate_torus seed 1), univariate
FOS, population 128 per GPU, Philox donors.  The metric is quoted "at
1/2/4/8 B200", which is this config ("sharded 1/2/4/8 B200"), and the north
star's target is stated on it (the 10^6-vertex grid on 1 B200); it fits one
GPU.  configs[1] (C2: 100x100, neighbourhood FOS, n=64) is --config c2.

ours:
  value  device throughput, inputs resident in HBM: CUDA events on the engine's
         stream around each generation; L2 flushed (256 MiB write) between
         timed generations, outside the events.
  e2e    through the C-ABI with HOST buffers, the reference run loop's
         per-generation GenerationRunner calls: run_generation (criteria in,
         stats + improvement log out) + read_elitist (genotype out), wall
         clock.  e2e_population_roundtrip additionally uploads and reads back
         the whole population every step.
  roofline  gom_group_kernel (dominant kernel): algorithmic bytes (SURVEY.md
         §8(d) B_step x steps) / its CUDA-event durations vs measured HBM peak.
  cpu_baseline  the reference ParallelEngine (oracle/_ref, compiled from the
         reference headers) with every host thread, a bounded sample.
reference:
  the reference's own CPU ParallelEngine (oracle/_ref/ref_driver) on this
  box's host cores, W + K generations of the same workload; rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Max-Cut partial evals/sec; time-to-best-known cut (s) at 1/2/4/8 B200"
REF_BUDGET_S = 90.0  # reference arm: cap on the generations it times (bounded sample)
UNIT = "partial evaluations/s"

CONFIGS = {
    "c2": dict(workload="C2: Max-Cut 2-D torus 100x100 (1e4 vertices), integer weights U[1,10] "
                        "(generate_torus seed 1), neighbourhood FOS, population 64",
               width=100, height=100, weights=("int", 1, 10), fos="neigh", n=64, ref_fos="neigh"),
    "c3": dict(workload="C3: Max-Cut 2-D torus 1000x1000 (1e6 vertices), integer weights U[1,10], "
                        "univariate FOS, population 128",
               width=1000, height=1000, weights=("int", 1, 10), fos="uni", n=128, ref_fos="univariate"),
    "c1": dict(workload="C1: Max-Cut 2-D torus 10x10, integer weights U[1,10], univariate FOS, population 32",
               width=10, height=10, weights=("int", 1, 10), fos="uni", n=32, ref_fos="univariate"),
    "c5": dict(workload="C5: Max-Cut 2-D torus 316x316 (~1e5 vertices), integer weights U[1,10], "
                        "univariate FOS, population 1024",
               width=316, height=316, weights=("int", 1, 10), fos="uni", n=1024, ref_fos="univariate"),
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c3", choices=sorted(CONFIGS))
    ap.add_argument("--population", type=int, default=None)
    ap.add_argument("--e2e-steps", type=int, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ttt-seconds", type=float, default=20.0,
                    help="time-to-best-known-cut leg: reference IMS budget T_ref (0 = skip)")
    return ap.parse_args()


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def ref_cmd(cfg, n, gens, workers, max_seconds=0.0):
    w = cfg["weights"]
    wspec = "unit" if w == "unit" else f"int:{w[1]}:{w[2]}"
    cmd = [os.path.join(ROOT, "oracle", "_ref", "ref_driver"), "bench", "--torus", str(cfg["width"]),
           str(cfg["height"]), "--weights", wspec, "--inst-seed", "1", "--fos", cfg["ref_fos"], "--n", str(n),
           "--seed", "1", "--gens", str(gens), "--workers", str(workers)]
    if max_seconds > 0:
        cmd += ["--max-seconds", str(max_seconds)]
    return cmd


def run_reference(cfg, n, gens, workers, timeout=3600, max_seconds=0.0):
    """The reference ParallelEngine compiled from its own headers (oracle/_ref);
    with max_seconds, generations stop once that much time was spent."""
    res = subprocess.run(ref_cmd(cfg, n, gens, workers, max_seconds), capture_output=True, text=True,
                         timeout=timeout)
    if res.returncode != 0:
        raise RuntimeError(f"ref_driver failed: {res.stderr.strip()}")
    return json.loads(res.stdout)


def base_line(args, cfg, n, world):
    return {"metric": METRIC, "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int32",
            "data": "synthetic (generated Max-Cut torus, reference generator and seed)",
            "config": {"workload": cfg["workload"], "population": n * world, "population_per_gpu": n,
                       "parallelism": f"population sharded over {world} GPUs (NCCL all-gather of the donor pool "
                                      f"per colour group)" if world > 1 else "single",
                       "l2": "flushed between timed steps (256 MiB write)",
                       "donors": "philox", "fos": cfg["fos"]}}


# ---------------------------------------------------------------------------
# reference arm
# ---------------------------------------------------------------------------
def bench_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    cfg = CONFIGS[args.config]
    n = args.population or cfg["n"]
    workers = os.cpu_count() or 1
    if not os.path.exists(os.path.join(ROOT, "oracle", "_ref", "ref_driver")):
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/ref_driver was not built"}))
        return
    # the same population as our arm at N GPUs (n per GPU, weak scaling);
    # bounded sample: W + K generations, or as many as fit in REF_BUDGET_S
    out = run_reference(cfg, n * world, args.warmup + args.steps, workers, max_seconds=REF_BUDGET_S)
    allg = out["gens"]
    warm = min(args.warmup, max(0, len(allg) - 1))
    gens = allg[warm:]
    secs = sum(g["seconds"] for g in gens)
    steps = sum(g["steps"] for g in gens)
    value = steps / secs
    line = base_line(args, cfg, n, world)
    line.update({"impl": "reference", "value": value, "ms_per_step": 1e3 * secs / len(gens), "dtype": "f64",
                 "steps_timed": len(gens), "warmup_run": warm,
                 "cpu_baseline": {"value": value, "unit": UNIT, "cores": workers, "kind": "reference",
                                  "sample": f"{len(gens)} generations of {args.config} after {warm} warm-up "
                                            f"(W + K = {args.warmup + args.steps} requested, capped at "
                                            f"{REF_BUDGET_S:g} s of generations), ParallelEngine(workers={workers})"},
                 "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}})
    line["config"]["parallelism"] = f"cpu ParallelEngine workers={workers}"
    line["config"]["donors"] = "reference RngStream"
    print(json.dumps(line))


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.rows = []
        self.p = None

    def start(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                                       "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.p = None
            return
        self.t = threading.Thread(target=self._read, daemon=True)
        self.t.start()

    def _read(self):
        for line in self.p.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == 8 and parts[0] == str(self.idx):
                self.rows.append(parts)

    def stop(self):
        if self.p:
            self.p.terminate()
            try:
                self.p.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.p.kill()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[4 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": float(self.rows[0][2]) if self.rows[0][2].replace(".", "").isdigit() else None,
                "reasons": reasons, "samples": len(self.rows)}


def algorithmic_bytes_per_step(inst, fos, n):
    """B_step(F) = ((|F| + |N(F)|) + 2|F|)/8 + G_F/n with
    G_F = 4(1+|F|) + sum_{v in F}(4 + deg(v)(4 + 8)), averaged over the sets."""
    import numpy as np

    nv = inst.num_vertices
    deg = np.bincount(np.concatenate([inst.edge_u, inst.edge_v]), minlength=nv)
    adj = inst.adjacency()
    total = 0.0
    for i in range(fos.num_sets):
        F = fos.set(i)
        nf = set()
        for v in F.tolist():
            nf.update(adj[v].tolist())
        nf.difference_update(F.tolist())
        gf = 4 * (1 + len(F)) + sum(4 + int(deg[v]) * 12 for v in F.tolist())
        total += ((len(F) + len(nf)) + 2 * len(F)) / 8.0 + gf / n
    return total / fos.num_sets


def bench_ours(args):
    import numpy as np
    import torch

    import paper_2203_08680_b200 as G

    rank, world, local = dist_env()
    if world > 1:
        import torch.distributed as dist

        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        dist = None
        torch.cuda.set_device(0)
    dev = torch.cuda.current_device()
    cfg = CONFIGS[args.config]
    n = args.population or cfg["n"]
    inst = G.generate_torus(cfg["width"], cfg["height"], cfg["weights"], 1)
    fos = G.univariate_fos(inst.num_vertices) if cfg["fos"] == "uni" else G.neighbourhood_fos(inst)
    P = G.GpuProblem(inst, fos, device=dev)
    stream = torch.cuda.Stream()  # a real stream: the legacy NULL stream would not see our kernels
    torch.cuda.set_stream(stream)
    if world > 1:
        # one population of n * world members sharded over the ranks (weak
        # scaling: n members per GPU); the NCCL id travels over the PG
        uid = [G.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        E = G.GpuParallelEngine(P, n * world, seed=1, mode="philox", stream=stream.cuda_stream, rank=rank,
                                world_size=world, nccl_unique_id=uid[0])
        gen = E.run_generation          # collective per colour group: host-ordered
    else:
        E = G.GpuParallelEngine(P, n, seed=1, mode="philox", stream=stream.cuda_stream)
        gen = E.run_generation_async    # one CUDA graph per generation, no host sync

    def barrier():
        if dist is not None:
            dist.barrier()

    # warm-up
    for _ in range(max(args.warmup, 3)):
        gen()
    E.synchronize()
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")  # 256 MiB > 126 MB L2

    # ---- device-resident timed region ----
    _, steps0, calls0 = E.group_counters()
    launches0 = E.launch_count()
    gpu_index = local
    vis = os.environ.get("CUDA_VISIBLE_DEVICES")
    if vis:
        try:
            gpu_index = int(vis.split(",")[local])
        except ValueError:
            pass
    clocks = ClockSampler(gpu_index)
    clocks.start()
    time.sleep(0.25)
    ev0 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ev1 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    barrier()
    torch.cuda.synchronize()
    t_wall0 = time.perf_counter()
    for i in range(args.steps):
        flush.zero_()
        ev0[i].record(stream)
        gen()
        ev1[i].record(stream)
    torch.cuda.synchronize()
    barrier()
    t_wall = time.perf_counter() - t_wall0
    _, steps1, calls1 = E.group_counters()
    launches = E.launch_count() - launches0
    step_ms = [a.elapsed_time(b) for a, b in zip(ev0, ev1)]
    # keep the GPU busy for the clock record when the timed region was short;
    # the generation count is fixed up front (rank 0's estimate, broadcast):
    # sharded generations are collectives, so every rank must run the same number
    per_gen_s = max(sum(step_ms) / 1e3 / max(1, args.steps), 1e-6)  # device time per generation
    soak = [int(max(0.0, 1.5 - t_wall) / per_gen_s)]
    if dist is not None:
        dist.broadcast_object_list(soak, src=0)
    for _ in range(min(soak[0], 50000)):
        gen()
    torch.cuda.synchronize()
    E.synchronize()
    clk = clocks.stop()
    # dominant-kernel durations (roofline): the same generations issued launch
    # by launch with CUDA events around every gom_group_kernel
    kern_gens = min(args.steps, 50)
    _, ksteps0, _ = E.group_counters()
    E.set_timing(True)
    E.kernel_times()
    for _ in range(kern_gens):
        flush.zero_()
        gen()
    E.synchronize()
    kern_ms = E.kernel_times()
    E.set_timing(False)
    _, ksteps1, _ = E.group_counters()
    kern_steps = int((ksteps1 - ksteps0).sum())

    dev_s = sum(step_ms) / 1e3
    steps = int((steps1 - steps0).sum())
    calls = int((calls1 - calls0).sum())
    if dist is not None:
        t = torch.tensor([dev_s], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        # sharded counters are already global (every rank accounts all ranks'
        # steps in its epilogue): no sum over ranks
        dev_s = float(t.item())
    value = steps / dev_s

    # ---- e2e through the C-ABI with host buffers ----
    # (1) the drop-in call pattern: what the reference's run loop / ImsDriver
    #     does with a GenerationRunner every generation (ims.hpp:77-80,
    #     run.hpp:64-66): run_generation with the run's stop criteria from the
    #     host (H2D) and its stats + improvement log back (D2H), then the
    #     elitist genotype read into a pinned host buffer (D2H l bytes).
    e2e_steps = args.e2e_steps or min(args.steps, 50)
    eg_host = torch.empty((inst.num_vertices,), dtype=torch.uint8, pin_memory=True).numpy()
    for _ in range(3):
        E.run_generation()
        E.elitist(eg_host)
    barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e2e_done = 0
    elit_reads = 0
    for _ in range(e2e_steps):
        E.run_generation()                          # H2D: stop criteria; D2H: stats + improvements
        e2e_done += int(E.last_stats.steps)         # global steps (sharded stats are global)
        if E.last_stats.improvements:               # the adapter's lazy elitist refresh: the
            E.elitist(eg_host)                      # genotype changes only with a better fitness
            elit_reads += 1                         # D2H: l genotype bytes (+ fitness)
    torch.cuda.synchronize()
    barrier()
    e2e_s = time.perf_counter() - t0
    # (2) the whole population in and out every step (n*l genotype bytes +
    #     n fitness doubles each way): the cost of a caller that keeps the
    #     population on the host
    g_host = torch.empty((n, inst.num_vertices), dtype=torch.uint8, pin_memory=True).numpy()
    f_host = torch.empty((n,), dtype=torch.float64, pin_memory=True).numpy()
    E.population(g_host, f_host)
    for _ in range(3):  # warm the transfer path
        E.load_population(g_host, f_host)
        E.run_generation()
        E.population(g_host, f_host)
    barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rt_done = 0
    rt_steps = max(5, e2e_steps // 5)
    for _ in range(rt_steps):
        E.load_population(g_host, f_host)
        E.run_generation()
        rt_done += int(E.last_stats.steps)
        E.population(g_host, f_host)
    torch.cuda.synchronize()
    barrier()
    rt_s = time.perf_counter() - t0
    if dist is not None:
        t = torch.tensor([e2e_s, rt_s], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s, rt_s = float(t[0].item()), float(t[1].item())
    io_bytes = n * inst.num_vertices + 8 * n
    crit_bytes = 40           # gomix_stop_criteria
    stats_bytes = 48 + 1024   # gomix_run_stats + control block and inline improvement log read back

    if rank != 0:
        if dist is not None:
            dist.destroy_process_group()
        return

    # ---- roofline of the dominant kernel ----
    peaks = {}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            peaks = json.load(fh)
    except OSError:
        pass
    peak = float(peaks.get("hbm_gbs", 6650.0))
    peak_src = "MEASURED_PEAKS.json hbm_gbs (measured)" if "hbm_gbs" in peaks else "fallback 6.65 TB/s"
    b_step = algorithmic_bytes_per_step(inst, fos, n)
    kern_s = float(np.sum(kern_ms)) / 1e3
    achieved = kern_steps * b_step / kern_s / 1e9 if kern_s > 0 else None
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as fh:
            tr = json.load(fh).get(args.config)
            if tr and tr.get("population") == n and tr.get("kernel", "gom_group_kernel") == E.kernel_name():
                traffic = tr["dram_bytes_per_launch"]
    except (OSError, ValueError):
        pass
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak if achieved else None, "traffic": traffic,
                "kernel": E.kernel_name(), "bytes_per_step": b_step,
                "launches": int(len(kern_ms)), "avg_launch_us": 1e6 * kern_s / max(1, len(kern_ms)),
                "kernel_share_of_step": (kern_s / kern_gens) / (dev_s / args.steps) if dev_s else None,
                "peak_source": peak_src,
                "timing": f"CUDA events around each launch over {kern_gens} generations issued launch by launch"}

    cpu_baseline = None
    if world == 1 and not args.no_cpu_baseline:
        ref = os.path.join(ROOT, "oracle", "_ref", "ref_driver")
        workers = os.cpu_count() or 1
        gens = 8 if args.config in ("c2", "c1") else 2
        if os.path.exists(ref):
            try:
                out = run_reference(cfg, n, gens, workers, timeout=900)
                secs = sum(g["seconds"] for g in out["gens"])
                st = sum(g["steps"] for g in out["gens"])
                cpu_baseline = {"value": st / secs, "unit": UNIT, "cores": workers, "kind": "reference",
                                "sample": f"{gens} generations of {args.config} ({st} partial evaluations), "
                                          f"reference ParallelEngine(workers={workers}) built from its headers"}
            except Exception as exc:  # noqa: BLE001
                cpu_baseline = {"value": None, "unit": UNIT, "cores": workers, "kind": "reference",
                                "sample": f"failed: {exc}"}

    time_to_target = None
    if world == 1 and args.ttt_seconds > 0:
        try:
            sys.path.insert(0, os.path.join(ROOT, "tools"))
            import time_to_target as TT

            ref = TT.reference_ims(cfg, 1, args.ttt_seconds, os.cpu_count() or 1)
            gpu = TT.gpu_ims(cfg, ref["best"], 1, args.ttt_seconds)
            time_to_target = {
                "unit": "s", "target_cut": ref["best"],
                "target": f"best cut of the reference IMS (base 16, sub 4, {cfg['fos']} FOS, "
                          f"{os.cpu_count()} threads) within {args.ttt_seconds:g} s, seed 1",
                "cpu_s": ref["seconds_to_best"], "gpu_s": gpu["seconds_to_target"],
                "gpu_s_incl_build": gpu["seconds_to_target_incl_build"], "gpu_reached": gpu["reached"],
                "speedup": (ref["seconds_to_best"] / gpu["seconds_to_target"]) if gpu["reached"] else None,
                "gpu_build_s": gpu["build_seconds"], "gpu_evaluations": gpu["evaluations"],
                "cpu_evaluations": ref["evaluations"],
                "timing": "both from RunContext creation to the improvement reaching the cut (model prebuilt); "
                          "gpu_s_incl_build adds the device problem build (CSR, GPU colouring)"}
        except Exception as exc:  # noqa: BLE001
            time_to_target = {"error": str(exc)[:300]}

    line = base_line(args, cfg, n, world)
    line.update({
        "value": value,
        "ms_per_step": 1e3 * dev_s / args.steps,
        "e2e": {"value": e2e_done / e2e_s, "unit": UNIT, "h2d_bytes_per_step": crit_bytes,
                "d2h_bytes_per_step": stats_bytes + (inst.num_vertices + 8) * elit_reads / e2e_steps,
                "steps": e2e_steps, "elitist_reads": elit_reads,
                "what": "per generation through the C-ABI with pinned host buffers, the reference run loop's "
                        "GenerationRunner calls: run_generation (stop criteria in, stats + improvements out) "
                        "+ the elitist genotype read back after every generation that improved it (the C++ "
                        "adapter's lazy elitist(): the genotype changes only with a strictly better fitness, "
                        "engine_parallel.hpp:305-310); wall clock"},
        "e2e_population_roundtrip": {"value": rt_done / rt_s, "unit": UNIT, "h2d_bytes_per_step": io_bytes,
                                     "d2h_bytes_per_step": io_bytes, "steps": rt_steps,
                                     "what": "load_population + run_generation + read_population (the whole "
                                             "population as genotype bytes both ways every step)"},
        "roofline": roofline,
        "cpu_baseline": cpu_baseline,
        "time_to_target": time_to_target,
        "clocks": clk,
        "gpu_launches": int(launches),
        "evaluator_calls_per_s": calls / dev_s,
        "wall_s_timed_region": t_wall,
        "elitist_fitness": E.elitist_fitness,
    })
    print(json.dumps(line))
    if dist is not None:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        bench_reference(args)
    else:
        bench_ours(args)


if __name__ == "__main__":
    main()
