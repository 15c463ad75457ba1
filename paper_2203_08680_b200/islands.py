"""Interleaved multistart over several GPUs (one process per GPU).

The reference runs one ImsDriver on one host (ims.hpp:38-101, run.hpp:72-82);
its populations are small (16, 32, 64, ...), so sharding each of them over
GPUs would leave every GPU a few solutions.  Across GPUs this module runs one
IMS per rank instead — an island model — and keeps the reference's exchange
rule between them: the run-wide best is offered to a population before its
generation and collected after it (ims.hpp:77-80), where "run-wide" now spans
the ranks.  Every `exchange_every` IMS steps the ranks all-reduce (max) their
best fitness and stop flag; when the global best improved, its owner (the
lowest rank holding it) broadcasts the genotype and every other rank offers it
to its smallest population (offer_elitist adopts iff strictly better,
engine_parallel.hpp:320-322) and collects it into its device-side best.

Rank 0 uses the run seed itself, so one rank is exactly ``run_gpu`` with IMS;
rank r > 0 uses ``mix64(seed + r)`` as its run seed (disjoint population
seeds through population_seed, run.hpp:36-39).  Stop criteria are evaluated
per rank (target, wall clock, the rank's own evaluation budget); any rank's
stop ends the run for all at the next exchange.
"""
from __future__ import annotations

import math
import time
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from .engine import GpuProblem, RecordingSink, RunContext, TerminationConfig, mix64
from .ims import GpuImsDriver, ImsConfig, _require_termination


class BestExchange:
    """Collective exchange of the run-wide best over torch.distributed (NCCL
    on GPUs, gloo on CPU).  All ranks call every method in the same order."""

    def __init__(self, num_vertices: int, device=None, group=None):
        import torch
        import torch.distributed as dist

        self.torch, self.dist = torch, dist
        self.nv = int(num_vertices)
        self.device = device if device is not None else "cpu"
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.shared_fit = -math.inf  # the best every rank has already received

    def exchange(self, local_fit: Optional[float], local_stop: bool, genotype_fn):
        """-> (global best fitness, global stop, genotype or None).  The
        genotype is returned (on every rank) only when the global best
        improved since the last exchange; genotype_fn() gives this rank's best
        genotype (uint8, num_vertices) and is only called on the owner."""
        torch, dist = self.torch, self.dist
        f = -math.inf if local_fit is None else float(local_fit)
        t = torch.tensor([f, 1.0 if local_stop else 0.0], dtype=torch.float64, device=self.device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=self.group)
        g_fit, g_stop = float(t[0].item()), bool(t[1].item() > 0)
        geno = None
        if g_fit > self.shared_fit:
            owner = torch.tensor([self.rank if f == g_fit else self.world], dtype=torch.int64, device=self.device)
            dist.all_reduce(owner, op=dist.ReduceOp.MIN, group=self.group)
            src = int(owner.item())
            buf = torch.empty(self.nv, dtype=torch.uint8, device=self.device)
            if self.rank == src:
                buf.copy_(torch.from_numpy(np.ascontiguousarray(genotype_fn(), np.uint8)))
            dist.broadcast(buf, src=dist.get_global_rank(self.group, src) if self.group is not None else src,
                           group=self.group)
            geno = buf.cpu().numpy()
            self.shared_fit = g_fit
        return g_fit, g_stop, geno

    def gather(self, obj):
        out = [None] * self.world
        self.dist.all_gather_object(out, obj, group=self.group)
        return out


@dataclass
class IslandResult:
    best_fitness: Optional[float] = None
    reason: str = "none"
    seconds_to_target: Optional[float] = None   # first rank to reach the target (common clock start)
    rank_seconds_to_target: List[Optional[float]] = field(default_factory=list)
    evaluations: float = 0.0                    # summed over ranks (gray-box units)
    rank_evaluations: List[float] = field(default_factory=list)
    populations: List[int] = field(default_factory=list)
    seconds: float = 0.0                        # until every rank stopped (max over ranks)
    exchanges: int = 0
    adopted: int = 0                            # genotypes this rank took from another rank


def run_islands(problem: GpuProblem, termination: TerminationConfig, seed: int = 1,
                ims: Optional[ImsConfig] = None, exchange: Optional[BestExchange] = None,
                exchange_every: int = 4, mode: str = "philox", **engine_kw) -> IslandResult:
    """One IMS per rank with the run-wide best exchanged between ranks (module
    docstring).  exchange None = a single rank (plain IMS).  Every rank's
    clock starts when its RunContext is created; callers put a barrier right
    before the call so the clocks start together."""
    _require_termination(termination)
    rank = exchange.rank if exchange else 0
    run_seed = seed if rank == 0 else mix64((seed + rank) & ((1 << 64) - 1))
    sink = RecordingSink()
    ctx = RunContext(termination, problem.comparator(), problem.info.num_edges, sink)
    drv = GpuImsDriver.for_problem(ims or ImsConfig(), problem, ctx, run_seed, mode=mode, **engine_kw)
    res = IslandResult()
    it = 0
    alive = True
    while True:
        if alive:
            alive = drv.step()
        it += 1
        if exchange is None:
            if not alive:
                break
            continue
        if it % exchange_every:  # the same iterations on every rank: the exchange is collective
            continue
        _, fit = drv.best.read(genotype=False)
        g_fit, g_stop, geno = exchange.exchange(fit, not alive, lambda: drv.best.read()[0])
        res.exchanges += 1
        if geno is not None and (fit is None or g_fit > fit) and alive and drv.runners:
            # ImsDriver's offer / collect with the other ranks' best
            if drv.runners[0].offer_elitist(geno, g_fit):
                drv.best.collect(drv.runners[0])
                res.adopted += 1
        if g_stop:
            if alive:
                ctx.control.request_stop("peer-stopped")
            break
    target = termination.target_fitness
    t_hit = None
    if target is not None:
        t_hit = next((r.seconds for r in sink.rows if problem.comparator().better(r.fitness, target)
                      or problem.comparator().equal(r.fitness, target)), None)
    _, best = drv.best.read(genotype=False)
    mine = {"t_hit": t_hit, "evals": ctx.control.evaluations(), "pops": drv.num_populations(),
            "secs": ctx.control.elapsed_seconds(), "best": best, "reason": ctx.control.reason}
    rows = exchange.gather(mine) if exchange else [mine]
    hits = [r["t_hit"] for r in rows]
    res.rank_seconds_to_target = hits
    res.seconds_to_target = min((h for h in hits if h is not None), default=None)
    res.rank_evaluations = [r["evals"] for r in rows]
    res.evaluations = float(sum(res.rank_evaluations))
    res.populations = [r["pops"] for r in rows]
    res.seconds = max(r["secs"] for r in rows)
    bests = [r["best"] for r in rows if r["best"] is not None]
    res.best_fitness = max(bests) if bests else None
    reasons = [r["reason"] for r in rows if r["reason"] not in ("none", "peer-stopped")]
    res.reason = "target-reached" if "target-reached" in reasons else (reasons[0] if reasons else ctx.control.reason)
    return res
