#!/usr/bin/env python3
"""Benchmark of the B200 GOM engine on BASELINE.json's headline metric.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c2]

One step = one GOM generation (ParallelEngine::run_generation,
engine_parallel.hpp:283-316) of the workload; the unit of work is one partial
evaluation = one executed (solution, linkage set) GOM step
(RunResult::GroupCounter::steps, runtime.hpp:170-175).

Default workload: BASELINE.json configs[2] = C3, Max-Cut 2-D torus 1000x1000
(10^6 vertices), integer weights U[1,10] (generate_torus seed 1), univariate
FOS, population 128, Philox donors.  The metric is quoted "at 1/2/4/8 B200",
which is this config ("population 128, sharded 1/2/4/8 B200"), and the north
star's target is stated on it (the 10^6-vertex grid on 1 B200); it fits one
GPU.  configs[1] (C2: 100x100, neighbourhood FOS, n=64) is --config c2.

Scaling: --scaling strong (default) keeps BASELINE's population of 128 in
total and shards it over the N GPUs (128/N members each, NCCL exchange per
colour group); --scaling weak gives every GPU 128 members.

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
REF_BUDGET_S = 900.0  # reference arm: safety cap on its W + K generations (C3: ~12 s each on 16 threads)
# time-to-target leg: a FIXED cut per config (from the reference's own IMS
# runs, tools/success_rate.py pilots), so every run and every N aim at the
# same value; the CPU reference is timed to it in the same run
TTT_TARGETS = {"c1": 1110.0, "c2": 103400.0, "c3": 9600000.0, "c5": None}
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
    ap.add_argument("--ttt-seconds", type=float, default=60.0,
                    help="time-to-target leg: wall budget of the reference IMS and of ours (0 = skip)")
    ap.add_argument("--transport", default=None, choices=["peer", "nccl"],
                    help="N > 1: exchanges over peer memory inside the kernels (default for univariate FOS) or NCCL")
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"],
                    help="strong: BASELINE's population in total over the N GPUs; weak: that many per GPU")
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


def population_total(args, cfg, world):
    """BASELINE C3 is "population 128, sharded 1/2/4/8 B200": strong scaling
    keeps the population fixed; weak scaling gives every GPU that many."""
    n = args.population or cfg["n"]
    return n if args.scaling == "strong" else n * world


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def base_line(args, cfg, n_total, world):
    return {"metric": METRIC, "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "int32",
            "data": "synthetic (generated Max-Cut torus, reference generator and seed)",
            "config": {"workload": cfg["workload"], "population": n_total, "population_per_gpu": n_total // world,
                       "parallelism": f"population sharded over {world} GPUs ({n_total // world} members each; "
                                      f"exchange of fitness / hashes / counters per colour group, row presence "
                                      f"per generation)" if world > 1 else "single",
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
    n_total = population_total(args, cfg, world)
    workers = os.cpu_count() or 1
    if not os.path.exists(os.path.join(ROOT, "oracle", "_ref", "ref_driver")):
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/ref_driver was not built"}))
        return
    # the same population and workload as our arm at N GPUs; one step = one
    # generation, W + K of them (a safety cap of REF_BUDGET_S s of
    # generations; steps reports how many were timed)
    out = run_reference(cfg, n_total, args.warmup + args.steps, workers, max_seconds=REF_BUDGET_S)
    allg = out["gens"]
    warm = min(args.warmup, max(0, len(allg) - 1))
    gens = allg[warm:]
    secs = sum(g["seconds"] for g in gens)
    steps = sum(g["steps"] for g in gens)
    value = steps / secs
    line = base_line(args, cfg, n_total, world)
    line.update({"impl": "reference", "value": value, "ms_per_step": 1e3 * secs / len(gens), "dtype": "f64",
                 "steps": len(gens), "steps_requested": args.steps, "warmup": warm,
                 "cpu_baseline": {"value": value, "unit": UNIT, "cores": workers, "kind": "reference",
                                  "cpu": cpu_model(),
                                  "sample": f"{len(gens)} generations of {args.config} after {warm} warm-up "
                                            f"generations, ParallelEngine(workers={workers}) built from the "
                                            f"reference headers (oracle/_ref/ref_driver)"},
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


def make_engine(G, P, n_total, seed, stream, rank, world, uid, transport):
    """One population of n_total members: single GPU, or sharded over the
    ranks (rank r holds n_total / world; transport "peer": exchanges inside
    the GOM kernels over peer memory, "nccl": NCCL calls between launches)."""
    if world > 1:
        return G.GpuParallelEngine(P, n_total, seed=seed, mode="philox", stream=stream.cuda_stream, rank=rank,
                                   world_size=world, nccl_unique_id=uid, transport=transport)
    return G.GpuParallelEngine(P, n_total, seed=seed, mode="philox", stream=stream.cuda_stream)


def bench_ours(args):
    import numpy as np
    import torch

    import paper_2203_08680_b200 as G

    rank, world, local = dist_env()
    if world > 1:
        import torch.distributed as dist

        # the communicators' set-up lines (ranks, devices, NVLS / P2P
        # transports) on stderr, so a run shows how many ranks took part
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        if os.environ.get("GOMIX_BENCH_ONE_GPU"):
            # code-path check on a one-GPU box: every rank on cuda:0, gloo for
            # the host plumbing (NCCL refuses two ranks on one device); the
            # peer transport itself works within a device (CUDA IPC)
            local = 0
            torch.cuda.set_device(0)
            dist.init_process_group("gloo")
        else:
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        dist = None
        torch.cuda.set_device(0)
    dev = torch.cuda.current_device()
    cfg = CONFIGS[args.config]
    n_total = population_total(args, cfg, world)
    if n_total % world:
        raise SystemExit(f"population {n_total} is not divisible by {world} GPUs")
    inst = G.generate_torus(cfg["width"], cfg["height"], cfg["weights"], 1)
    fos = G.univariate_fos(inst.num_vertices) if cfg["fos"] == "uni" else G.neighbourhood_fos(inst)
    P = G.GpuProblem(inst, fos, device=dev)
    stream = torch.cuda.Stream()  # a real stream: the legacy NULL stream would not see our kernels
    torch.cuda.set_stream(stream)
    uid = None
    # univariate FOS (C1/C3/C5): the peer transport — every exchange inside
    # the GOM kernels over NVLink peer memory, generations queued as CUDA
    # graphs; other FOS: NCCL between launches, host-ordered
    transport = args.transport or ("peer" if cfg["fos"] == "uni" else "nccl")
    if world > 1 and transport == "nccl":  # the NCCL id travels over the process group
        box = [G.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(box, src=0)
        uid = box[0]
    E = make_engine(G, P, n_total, 1, stream, rank, world, uid, transport)
    queued = world == 1 or transport == "peer"
    gen = E.run_generation_async if queued else E.run_generation

    def barrier():
        if dist is not None:
            dist.barrier()

    def max_over_ranks(*xs):
        if dist is None:
            return xs
        t = torch.tensor(list(xs), dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return tuple(float(v) for v in t.tolist())

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
    # by launch with CUDA events around every GOM kernel launch
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
    # sharded counters are already global (every rank accounts all ranks'
    # steps in its epilogue): no sum over ranks, the time is the max
    (dev_s,) = max_over_ranks(dev_s)
    value = steps / dev_s

    # ---- active phase: generations 1-5 of a fresh population ----
    # (the timed generations above are the steady state, where most pairs are
    # neutral or rejected; early generations accept and improve far more)
    E_act = make_engine(G, P, n_total, 2, stream, rank, world, uid, transport)
    act_gens = 5
    a0 = [torch.cuda.Event(enable_timing=True) for _ in range(act_gens)]
    a1 = [torch.cuda.Event(enable_timing=True) for _ in range(act_gens)]
    _, as0, _ = E_act.group_counters()
    barrier()
    torch.cuda.synchronize()
    for i in range(act_gens):
        flush.zero_()
        a0[i].record(stream)
        (E_act.run_generation_async if queued else E_act.run_generation)()
        a1[i].record(stream)
    torch.cuda.synchronize()
    E_act.synchronize()
    _, as1, _ = E_act.group_counters()
    (act_s,) = max_over_ranks(sum(x.elapsed_time(y) for x, y in zip(a0, a1)) / 1e3)
    act_steps = int((as1 - as0).sum())
    active = {"value": act_steps / act_s, "unit": UNIT, "generations": "1-5 of a fresh population (seed 2)",
              "ms_per_step": 1e3 * act_s / act_gens}
    del E_act

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
    n_local = n_total // world
    g_host = torch.empty((n_local, inst.num_vertices), dtype=torch.uint8, pin_memory=True).numpy()
    f_host = torch.empty((n_local,), dtype=torch.float64, pin_memory=True).numpy()
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
    e2e_s, rt_s = max_over_ranks(e2e_s, rt_s)
    io_bytes = n_local * inst.num_vertices + 8 * n_local
    crit_bytes = 40           # gomix_stop_criteria
    stats_bytes = 48 + 1024   # gomix_run_stats + control block and inline improvement log read back

    # ---- time to a fixed target cut (every rank: one IMS per GPU) ----
    time_to_target = None
    target = TTT_TARGETS.get(args.config)
    if args.ttt_seconds > 0 and target is not None:
        time_to_target = time_to_target_leg(args, cfg, G, P, inst, fos, target, rank, world, dist, dev)

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
    b_step = algorithmic_bytes_per_step(inst, fos, n_local)
    kern_s = float(np.sum(kern_ms)) / 1e3
    achieved = kern_steps / world * b_step / kern_s / 1e9 if kern_s > 0 else None  # this rank's share of the steps
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as fh:
            tr = json.load(fh).get(args.config)
            if tr and tr.get("population") == n_local and tr.get("kernel", "gom_group_kernel") == E.kernel_name():
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
                out = run_reference(cfg, n_total, gens + 1, workers, timeout=900)
                timed = out["gens"][1:]  # the first generation is the warm-up
                secs = sum(g["seconds"] for g in timed)
                st = sum(g["steps"] for g in timed)
                cpu_baseline = {"value": st / secs, "unit": UNIT, "cores": workers, "kind": "reference",
                                "cpu": cpu_model(),
                                "sample": f"generations 2-{gens + 1} of {args.config} ({st} partial evaluations) "
                                          f"after 1 warm-up generation, reference ParallelEngine(workers={workers}) "
                                          f"built from its headers"}
            except Exception as exc:  # noqa: BLE001
                cpu_baseline = {"value": None, "unit": UNIT, "cores": workers, "kind": "reference",
                                "sample": f"failed: {exc}"}

    line = base_line(args, cfg, n_total, world)
    if world > 1:
        line["config"]["transport"] = transport
    line.update({
        "value": value,
        "ms_per_step": 1e3 * dev_s / args.steps,
        "active_phase": active,
        "e2e": {"value": e2e_done / e2e_s, "unit": UNIT, "h2d_bytes_per_step": crit_bytes,
                "d2h_bytes_per_step": stats_bytes + (inst.num_vertices + 8) * elit_reads / e2e_steps,
                "steps": e2e_steps, "elitist_reads": elit_reads,
                "what": "per generation through the C-ABI with pinned host buffers, the reference run loop's "
                        "GenerationRunner calls: run_generation (stop criteria in, stats + improvements out) "
                        "+ the elitist genotype read back after every generation that improved it (the C++ "
                        "adapter's lazy elitist(): the genotype changes only with a strictly better fitness, "
                        "engine_parallel.hpp:305-310); wall clock, max over ranks"},
        "e2e_population_roundtrip": {"value": rt_done / rt_s, "unit": UNIT, "h2d_bytes_per_step": io_bytes,
                                     "d2h_bytes_per_step": io_bytes, "steps": rt_steps,
                                     "what": "load_population + run_generation + read_population (the whole "
                                             "population as genotype bytes both ways every step, per rank)"},
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


def time_to_target_leg(args, cfg, G, P, inst, fos, target, rank, world, dist, dev):
    """Time to a fixed cut: the reference's run_parallel IMS (rank 0, every
    host thread) and ours — one IMS per GPU with the run-wide best exchanged
    between them (paper_2203_08680_b200/islands.py; one GPU = run_gpu's IMS).
    Both clocks run from RunContext creation with the model prebuilt; every
    GPU rank starts after a barrier; the GPU time is the first rank to reach
    the cut."""
    import torch

    from paper_2203_08680_b200.islands import BestExchange, run_islands

    sys.path.insert(0, os.path.join(ROOT, "tools"))
    import time_to_target as TT

    cpu = None
    if rank == 0:
        try:
            cpu = TT.reference_to_target(cfg, 1, target, args.ttt_seconds, os.cpu_count() or 1)
        except Exception as exc:  # noqa: BLE001
            cpu = {"error": str(exc)[:300]}
    # the IMS population sizes' kernels load on first use: a one-time process
    # cost, paid here untimed on a tiny problem
    TT.warm_device()
    torch.cuda.synchronize()
    # the device model build, timed apart (CSR, colouring, plans): the median
    # of 3 builds, every sample reported (one build on a fresh box has varied
    # 0.05-0.18 s between runs)
    build_samples = []
    for _ in range(3):
        t0 = time.perf_counter()
        Pb = G.GpuProblem(inst, fos, device=dev)
        build_samples.append(time.perf_counter() - t0)
        del Pb
    build_s = sorted(build_samples)[1]
    ex = BestExchange(inst.num_vertices, device=torch.device("cuda", dev)) if world > 1 else None
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    r = run_islands(P, G.TerminationConfig(target_fitness=target, max_seconds=args.ttt_seconds), seed=1,
                    exchange=ex)
    if rank != 0:
        return None
    out = {"unit": "s", "target_cut": target,
           "target": f"fixed cut for {args.config} (tools/success_rate.py STUDY; the reference's IMS reaches it "
                     f"in most runs), seed 1, wall budget {args.ttt_seconds:g} s each side",
           "cpu": cpu, "cpu_s": (cpu or {}).get("seconds_to_target"),
           "gpu_s": r.seconds_to_target, "gpu_reached": r.reason == "target-reached",
           "gpu_rank_s": r.rank_seconds_to_target, "gpu_build_s": build_s, "gpu_build_samples_s": build_samples,
           "gpu_s_incl_build": (r.seconds_to_target + build_s) if r.seconds_to_target is not None else None,
           "gpu_evaluations": r.evaluations, "gpu_populations": r.populations,
           "gpu_exchanges": r.exchanges,
           "timing": "both from RunContext creation to the improvement reaching the cut (model prebuilt); "
                     "gpu_s_incl_build adds the device problem build (median of 3); N GPUs = one IMS per GPU with the best "
                     "exchanged (islands.py), time of the first rank to reach the cut"}
    if out["cpu_s"] and out["gpu_s"]:
        out["speedup"] = out["cpu_s"] / out["gpu_s"]
        out["speedup_incl_build"] = out["cpu_s"] / out["gpu_s_incl_build"]
    return out


def main():
    args = parse()
    if args.impl == "reference":
        bench_reference(args)
    else:
        bench_ours(args)


if __name__ == "__main__":
    main()
