"""Interleaved multistart (IMS) and whole runs on the B200 engine.

Mirrors the reference's host-side run API so time-to-target runs read like
its own:

* ``ImsConfig`` / ``GpuImsDriver``  — ``ImsDriver`` (ims.hpp:25-101): population
  i+1 is twice the size of population i and runs one generation per
  ``subgenerations`` generations of its predecessor; populations are created
  when the schedule first reaches them; the run-wide best is offered to a
  population right before each of its generations and collected after.  The
  best lives on the device (gomix_gpu_ims_collect / _offer): exchanging it
  costs no host round trip.
* ``run_gpu`` — ``detail::run_with<ParallelEngine>`` (run.hpp:41-97): a single
  population or IMS until a termination criterion fires; returns a
  ``RunResult`` (best, reason, evaluations, generations, populations).

Population seeds follow ``population_seed`` (run.hpp:36-39).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import _capi
from ._capi import check, lib
from .engine import GpuParallelEngine, GpuProblem, RunContext, TerminationConfig, TraceSink, population_seed


@dataclass
class ImsConfig:
    """ims.hpp:25-29."""
    base_population: int = 16
    subgenerations: int = 4
    max_populations: int = 0  # 0 = unlimited


@dataclass
class RunResult:
    """runtime.hpp:160-176 (the fields a run reports)."""
    best_fitness: Optional[float] = None
    best_genotype: Optional[np.ndarray] = None
    reason: str = "none"
    evaluations: float = 0.0
    generations: int = 0
    populations: int = 0
    seconds: float = 0.0
    group_steps: Optional[np.ndarray] = None
    group_calls: Optional[np.ndarray] = None


class DeviceBest:
    """ImsDriver::best_ kept on the problem's device."""

    def __init__(self, problem: GpuProblem):
        self.problem = problem
        h = C.c_void_p()
        check(lib().gomix_gpu_ims_best_create(problem.h, C.byref(h)))
        self.h = h
        self._destroy = lib().gomix_gpu_ims_best_destroy  # kept: module globals are gone at interpreter exit

    def __del__(self):
        if getattr(self, "h", None):
            self._destroy(self.h)
            self.h = None

    def collect(self, engine: GpuParallelEngine):
        check(lib().gomix_gpu_ims_collect(self.h, engine.h))

    def offer(self, engine: GpuParallelEngine):
        check(lib().gomix_gpu_ims_offer(self.h, engine.h))

    def read(self, genotype: bool = True):
        g = np.zeros(self.problem.info.num_vertices, np.uint8) if genotype else None
        f, v = C.c_double(), C.c_int32()
        check(lib().gomix_gpu_ims_best_read(self.h, _capi.ptr(g), C.byref(f), C.byref(v)))
        return (g, f.value) if v.value else (None, None)


class GpuImsDriver:
    """ImsDriver (ims.hpp:38-101).  ``factory(population_size, population_id)``
    builds a runner (RunnerFactory, ims.hpp:31-32); ``best`` exchanges the
    run-wide best (collect / offer).  ``for_problem`` wires the B200 engine and
    the device-resident best."""

    def __init__(self, cfg: ImsConfig, factory, ctx: RunContext, best):
        if cfg.base_population <= 0:
            raise ValueError("ims: base population must be positive")
        if cfg.subgenerations <= 0:
            raise ValueError("ims: subgeneration factor must be positive")
        self.cfg, self.factory, self.ctx, self.best = cfg, factory, ctx, best
        self.runners: List = []
        self.gens: List[int] = []

    @classmethod
    def for_problem(cls, cfg: ImsConfig, problem: GpuProblem, ctx: RunContext, seed: int, mode: str = "philox",
                    **engine_kw) -> "GpuImsDriver":
        """Populations seeded by population_seed(seed, id) (run.hpp:77)."""
        def factory(size, pop_id):
            return GpuParallelEngine(problem, size, population_seed(seed, pop_id), ctx=ctx, population_id=pop_id,
                                     mode=mode, **engine_kw)
        return cls(cfg, factory, ctx, DeviceBest(problem))

    def population_size(self, i: int) -> int:
        return self.cfg.base_population << i

    def num_populations(self) -> int:
        return len(self.runners)

    def step(self) -> bool:
        """Advance the smallest population one generation plus whatever larger
        populations fall due; False once the run has been stopped."""
        if self.ctx.control.stop_requested():
            return False
        self._advance(0)
        return not self.ctx.control.stop_requested()

    def _advance(self, i: int):
        ctl = self.ctx.control
        if ctl.stop_requested():
            return
        if i >= len(self.runners):
            if self.cfg.max_populations and len(self.runners) >= self.cfg.max_populations:
                return
            self.runners.append(self.factory(self.population_size(i), i + 1))
            self.gens.append(0)
            self.best.collect(self.runners[i])  # the fresh population's initial elitist counts
            if ctl.stop_requested():
                return
        r = self.runners[i]
        self.best.offer(r)
        r.run_generation()
        self.gens[i] += 1
        self.best.collect(r)
        if not ctl.stop_requested() and self.gens[i] % self.cfg.subgenerations == 0:
            self._advance(i + 1)


def _require_termination(t: TerminationConfig):
    if t.max_evaluations is None and t.max_seconds is None and t.target_fitness is None \
            and t.max_generations is None:
        raise ValueError("run: needs at least one termination criterion")


def run_gpu(problem: GpuProblem, termination: TerminationConfig, seed: int = 1, population_size: int = 64,
            use_ims: bool = True, ims: Optional[ImsConfig] = None, sink: Optional[TraceSink] = None,
            mode: str = "philox", ctx: Optional[RunContext] = None, **engine_kw) -> RunResult:
    """run_with<ParallelEngine> (run.hpp:41-97) on the B200 engine.  The
    run's clock starts when its RunContext is created (runtime.hpp:62-68)."""
    _require_termination(termination)
    ctx = ctx if ctx is not None else RunContext(termination, problem.comparator(), problem.info.num_edges, sink)
    res = RunResult()
    k = problem.num_groups
    steps = np.zeros(k, np.uint64)
    calls = np.zeros(k, np.uint64)
    if not use_ims:
        eng = GpuParallelEngine(problem, population_size, seed, ctx=ctx, mode=mode, **engine_kw)
        while not ctx.control.stop_requested():
            eng.run_generation()
        res.best_genotype, res.best_fitness = eng.elitist()
        res.generations = eng.generation()
        res.populations = 1
        _, st, ca = eng.group_counters()
        steps += st
        calls += ca
    else:
        drv = GpuImsDriver.for_problem(ims or ImsConfig(), problem, ctx, seed, mode=mode, **engine_kw)
        while drv.step():
            pass
        res.best_genotype, res.best_fitness = drv.best.read()
        res.generations = drv.runners[0].generation() if drv.runners else 0
        res.populations = drv.num_populations()
        for r in drv.runners:
            _, st, ca = r.group_counters()
            steps += st
            calls += ca
    res.reason = ctx.control.reason
    res.evaluations = ctx.control.evaluations()
    res.seconds = ctx.control.elapsed_seconds()
    res.group_steps, res.group_calls = steps, calls
    return res
