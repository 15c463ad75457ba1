"""Python face of the B200 GOM engine, mirroring the reference's engine API.

    reference (proj/include/gomix/)                here
    ModelArtifacts + groups (model.hpp:25-29)   -> GpuProblem
    ParallelEngine (engine_parallel.hpp:255)    -> GpuParallelEngine
    TerminationConfig/RunControl/RunContext     -> TerminationConfig / RunControl / RunContext
      (runtime.hpp:50-161)
    ImsDriver (ims.hpp:38-101), run_parallel    -> ImsDriver, run_parallel (run.py)

All compute goes through libgomix_b200.so (C-ABI, include/gomix_gpu.h); this
module only marshals arrays and keeps the run-wide bookkeeping the reference
keeps on the host.
"""
from __future__ import annotations

import ctypes as C
import time
from dataclasses import dataclass, field
from typing import Callable, List, Optional

import numpy as np

from . import _capi
from ._capi import check, lib
from .maxcut import Fos, MaxCutInstance


def mix64(x: int) -> int:
    """rng.hpp:11-16."""
    M = (1 << 64) - 1
    x = (x + 0x9E3779B97F4A7C15) & M
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & M
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & M
    return x ^ (x >> 31)


def population_seed(run_seed: int, population_id: int) -> int:
    """run.hpp:36-39."""
    return mix64((run_seed + 0x9E3779B97F4A7C15 * population_id) & ((1 << 64) - 1))


@dataclass
class FitnessComparator:
    """graybox.hpp:22-35."""
    exact: bool = True
    rel_tol: float = 1e-9

    def scale(self, a, b):
        return self.rel_tol * max(1.0, abs(a), abs(b))

    def better(self, a, b):
        return a > b if self.exact else a - b > self.scale(a, b)

    def equal(self, a, b):
        return a == b if self.exact else abs(a - b) <= self.scale(a, b)


# ---------------------------------------------------------------------------
# run bookkeeping (runtime.hpp)
# ---------------------------------------------------------------------------
@dataclass
class TerminationConfig:
    max_evaluations: Optional[float] = None  # gray-box units
    max_seconds: Optional[float] = None
    target_fitness: Optional[float] = None
    max_generations: Optional[int] = None


@dataclass
class TraceRecord:
    seconds: float
    evaluations: float
    generation: int
    population: int
    fitness: float


class RunControl:
    """runtime.hpp:60-123; evaluator calls are an exact integer count."""

    def __init__(self, cfg: TerminationConfig, cmp: FitnessComparator, num_subfunctions: int):
        self.cfg, self.cmp, self.q = cfg, cmp, num_subfunctions
        self.calls = 0
        self.stop = False
        self.reason = "none"
        self.start()

    def start(self):
        self._t0 = time.perf_counter()

    def elapsed_seconds(self):
        return time.perf_counter() - self._t0

    def evaluations(self):
        return 0.0 if self.q == 0 else self.calls / self.q

    def add_evaluator_calls(self, calls: int):
        self.calls += int(calls)
        if self.cfg.max_evaluations is not None and self.evaluations() >= self.cfg.max_evaluations:
            self.request_stop("evaluation-budget")

    def check_time(self):
        if not self.stop and self.cfg.max_seconds is not None and self.elapsed_seconds() >= self.cfg.max_seconds:
            self.request_stop("wall-clock")

    def note_best(self, fitness):
        t = self.cfg.target_fitness
        if not self.stop and t is not None and (self.cmp.better(fitness, t) or self.cmp.equal(fitness, t)):
            self.request_stop("target-reached")

    def stop_requested(self):
        return self.stop

    def request_stop(self, reason: str):
        if not self.stop:
            self.stop, self.reason = True, reason

    def criteria(self) -> _capi.StopCriteria:
        c = self.cfg
        return _capi.StopCriteria(c.max_evaluations is not None, c.max_evaluations or 0.0, self.calls,
                                  c.target_fitness is not None, c.target_fitness or 0.0)


class TraceSink:
    def improvement(self, rec: TraceRecord):
        pass

    def boundary(self, rec: TraceRecord):
        pass


class RecordingSink(TraceSink):
    def __init__(self):
        self.rows: List[TraceRecord] = []

    def improvement(self, rec):
        self.rows.append(rec)


class RunContext:
    """runtime.hpp:128-161: shared control, trace sink and monotone best."""

    def __init__(self, cfg: TerminationConfig, cmp: FitnessComparator, num_subfunctions: int,
                 sink: Optional[TraceSink] = None):
        self.control = RunControl(cfg, cmp, num_subfunctions)
        self.sink = sink
        self.cmp = cmp
        self.best: Optional[float] = None

    def report_improvement(self, fitness, generation, population):
        if self.best is not None and not self.cmp.better(fitness, self.best):
            return
        self.best = fitness
        self.control.note_best(fitness)
        if self.sink:
            self.sink.improvement(TraceRecord(self.control.elapsed_seconds(), self.control.evaluations(),
                                              generation, population, fitness))

    def report_boundary(self, fitness, generation, population):
        self.control.check_time()
        if not self.sink:
            return
        if self.best is not None and self.cmp.better(self.best, fitness):
            fitness = self.best
        self.sink.boundary(TraceRecord(self.control.elapsed_seconds(), self.control.evaluations(),
                                       generation, population, fitness))


# ---------------------------------------------------------------------------
# problem (shared model) and engine (one population)
# ---------------------------------------------------------------------------
class GpuProblem:
    """Device-resident instance + FOS + GPU Welsh-Powell colour groups + plans.
    colour: optional prebuilt ColorGroups as one colour per set (adopted like
    EngineConfig::fixed_model, engine_parallel.hpp:271-272)."""

    def __init__(self, instance: MaxCutInstance, fos: Fos, colour=None, device: int = 0):
        self.instance, self.fos = instance, fos
        L = lib()
        h = C.c_void_p()
        col = None if colour is None else np.ascontiguousarray(colour, np.int32)
        check(L.gomix_gpu_problem_create(C.byref(instance._struct()), C.byref(fos._struct()),
                                         _capi.ptr(col), device, C.byref(h)))
        self.h = h
        self._destroy = L.gomix_gpu_problem_destroy  # kept: module globals are gone at interpreter exit
        info = _capi.ProblemInfo()
        check(L.gomix_gpu_problem_info(self.h, C.byref(info)))
        self.info = info
        k = info.num_groups
        off = np.zeros(k + 1, np.uint64)
        sets = np.zeros(info.num_sets, np.uint64)
        check(L.gomix_gpu_problem_groups(self.h, off.ctypes.data, sets.ctypes.data))
        self.group_offset, self.group_sets = off, sets
        fp = np.zeros(info.num_sets, np.uint64)
        check(L.gomix_gpu_problem_footprints(self.h, fp.ctypes.data))
        self.footprints = fp

    def __del__(self):
        if getattr(self, "h", None):
            self._destroy(self.h)
            self.h = None

    @property
    def num_groups(self) -> int:
        return int(self.info.num_groups)

    @property
    def groups(self):
        o = self.group_offset
        return [self.group_sets[o[c]:o[c + 1]] for c in range(self.num_groups)]

    def colour(self) -> np.ndarray:
        col = np.zeros(self.info.num_sets, np.int32)
        for c, g in enumerate(self.groups):
            col[g] = c
        return col

    @property
    def exact(self) -> bool:
        return bool(self.info.exact)

    def comparator(self) -> FitnessComparator:
        return FitnessComparator(self.exact)


class GpuParallelEngine:
    """ParallelEngine (engine_parallel.hpp:255-368) on a B200.

    mode "replay": init, group order and donors follow the reference's
    RngStream(seed) exactly (bit-identical populations); "philox": donors are
    drawn on the device from a counter-based stream (production)."""

    def __init__(self, problem: GpuProblem, population_size: int, seed: int = 1,
                 ctx: Optional[RunContext] = None, population_id: int = 1, mode: str = "replay",
                 record_batch: bool = False, ordered_float: bool = False, time_kernels: bool = False,
                 genotypes: Optional[np.ndarray] = None, stream=None, rank: int = 0, world_size: int = 1,
                 nccl_unique_id: Optional[bytes] = None, lane_per_solution: bool = False,
                 per_group_kernels: bool = False, truth_table: bool = True,
                 forced_improvement: bool = False, transport: str = "nccl", process_group=None):
        """world_size > 1: this process's shard of a population of
        `population_size` members over world_size GPUs (Philox mode); every
        rank calls run_generation / elitist collectively.  transport "nccl":
        every rank passes the same nccl_unique_id (see nccl_unique_id());
        "peer": the GOM kernels exchange over peer memory themselves
        (gom_peer.cuh; univariate variable-once FOS), the blocks' CUDA IPC
        handles are all-gathered over torch.distributed (process_group)."""
        if population_size <= 0:
            raise ValueError("engine: population must be non-empty")
        self.problem = problem
        self.n_global = int(population_size)
        self.world_size, self.rank = int(world_size), int(rank)
        self.n = self.n_global // max(1, self.world_size)
        self.pop_id = population_id
        self.ctx = ctx if ctx is not None else RunContext(TerminationConfig(), problem.comparator(),
                                                          problem.info.num_edges)
        flags = (_capi.FLAG_RECORD_BATCH if record_batch else 0) | (_capi.FLAG_ORDERED_FLOAT if ordered_float else 0) \
            | (_capi.FLAG_TIME_KERNELS if time_kernels else 0) \
            | (_capi.FLAG_LANE_PER_SOLUTION if lane_per_solution else 0) \
            | (_capi.FLAG_PER_GROUP_KERNELS if per_group_kernels else 0) \
            | (0 if truth_table else _capi.FLAG_NO_TRUTH_TABLE) \
            | (_capi.FLAG_FORCED_IMPROVEMENT if forced_improvement else 0) \
            | (_capi.FLAG_PEER_TRANSPORT if transport == "peer" and self.world_size > 1 else 0)
        self._nid = None if nccl_unique_id is None else C.create_string_buffer(bytes(nccl_unique_id), 128)
        cfg = _capi.EngineConfig(self.n_global, seed, _capi.MODE_REPLAY if mode == "replay" else _capi.MODE_PHILOX,
                                 flags, population_id, self.rank, self.world_size,
                                 None if self._nid is None else C.cast(self._nid, C.c_void_p))
        h = C.c_void_p()
        check(lib().gomix_gpu_engine_create(problem.h, C.byref(cfg), C.byref(h)))
        self.h = h
        self._destroy = lib().gomix_gpu_engine_destroy
        if transport == "peer" and self.world_size > 1:
            import torch.distributed as dist

            mine = C.create_string_buffer(_capi.PEER_HANDLE_BYTES)
            check(lib().gomix_gpu_peer_export(self.h, C.cast(mine, C.c_void_p)))
            every = [None] * self.world_size
            dist.all_gather_object(every, mine.raw, group=process_group)
            allh = C.create_string_buffer(b"".join(every), _capi.PEER_HANDLE_BYTES * self.world_size)
            check(lib().gomix_gpu_peer_connect(self.h, C.cast(allh, C.c_void_p)))
        if stream is not None:
            check(lib().gomix_gpu_set_stream(self.h, C.c_void_p(stream)))
        self._elitist_fitness = None
        g = None
        if genotypes is not None:
            g = np.ascontiguousarray(genotypes, np.uint8)
            if g.shape != (self.n, problem.info.num_vertices):
                raise ValueError("graybox: genotype shape mismatch")
        stats = _capi.RunStats()
        crit = self.ctx.control.criteria()
        check(lib().gomix_gpu_init_population(self.h, _capi.ptr(g), C.byref(crit), C.byref(stats)))
        self._absorb(stats, generation=0)

    def __del__(self):
        if getattr(self, "h", None):
            self._destroy(self.h)
            self.h = None

    # ---- bookkeeping shared with RunContext -----------------------------------
    def _absorb(self, stats: _capi.RunStats, generation: int):
        """Replay the call's accounting into the run-wide RunContext in the
        reference's order: evaluator calls up to each improvement, the
        improvement, then the rest (engine_parallel.hpp:298-310)."""
        ctl = self.ctx.control
        start = ctl.calls
        end = start + int(stats.evaluator_calls)
        fit, calls_at = self.improvements(int(stats.improvements)) if stats.improvements else ((), ())
        if stats.stopped and stats.stop_reason == 1:
            ctl.request_stop("evaluation-budget")
        for f, c in zip(list(fit), list(calls_at)):
            ctl.calls = max(ctl.calls, int(c))
            self.ctx.report_improvement(float(f), generation, self.pop_id)
        ctl.calls = end
        if stats.stopped:
            ctl.request_stop(_capi.STOP_NAMES[stats.stop_reason])
        self._elitist_fitness = float(stats.elitist_fitness)
        self.last_stats = stats

    def improvements(self, count: int):
        buf = np.zeros(max(count, 1), np.float64)
        calls = np.zeros(max(count, 1), np.uint64)
        got = C.c_uint64()
        check(lib().gomix_gpu_read_improvements(self.h, buf.ctypes.data, calls.ctypes.data, count, C.byref(got)))
        return buf[:got.value], calls[:got.value]

    # ---- GenerationRunner (ims.hpp:14-22) -----------------------------------------
    def run_generation(self):
        ctl = self.ctx.control
        if ctl.stop_requested():
            return
        mg = ctl.cfg.max_generations
        if mg is not None and self.generation() >= mg:
            ctl.request_stop("generation-limit")
            return
        gen = self.generation()
        stats = _capi.RunStats()
        crit = ctl.criteria()
        check(lib().gomix_gpu_run_generation(self.h, C.byref(crit), C.byref(stats)))
        self._absorb(stats, gen)
        if not stats.stopped:
            self.ctx.report_boundary(self._elitist_fitness, self.generation(), self.pop_id)

    def run_generation_async(self):
        """Queue one generation without a host sync (Philox mode, no stop
        criteria); the run-wide bookkeeping is not updated."""
        check(lib().gomix_gpu_run_generation_async(self.h))

    def synchronize(self) -> _capi.RunStats:
        stats = _capi.RunStats()
        check(lib().gomix_gpu_synchronize(self.h, C.byref(stats)))
        self._elitist_fitness = float(stats.elitist_fitness)
        return stats

    def load_population(self, genotypes: np.ndarray, fitness: Optional[np.ndarray] = None):
        g = np.ascontiguousarray(genotypes, np.uint8)
        if g.shape != (self.n, self.problem.info.num_vertices):
            raise ValueError("graybox: genotype shape mismatch")
        f = None if fitness is None else np.ascontiguousarray(fitness, np.float64)
        check(lib().gomix_gpu_load_population(self.h, g.ctypes.data, _capi.ptr(f)))

    def generation(self) -> int:
        g = C.c_int64()
        check(lib().gomix_gpu_generation(self.h, C.byref(g)))
        return g.value

    def elitist(self, genotype_out: Optional[np.ndarray] = None):
        """(genotype, fitness) of the elitist; an optional caller buffer (e.g.
        pinned host memory, num_vertices uint8) is filled in place."""
        g = genotype_out if genotype_out is not None else np.zeros(self.problem.info.num_vertices, np.uint8)
        assert g.dtype == np.uint8 and g.shape == (self.problem.info.num_vertices,) and g.flags.c_contiguous
        f = C.c_double()
        check(lib().gomix_gpu_read_elitist(self.h, g.ctypes.data, C.byref(f)))
        return g, f.value

    @property
    def elitist_fitness(self) -> float:
        return self._elitist_fitness

    def offer_elitist(self, genotype, fitness) -> bool:
        adopted = C.c_int32()
        g = np.ascontiguousarray(genotype, np.uint8)
        check(lib().gomix_gpu_offer_elitist(self.h, g.ctypes.data, float(fitness), C.byref(adopted)))
        if adopted.value:
            self._elitist_fitness = float(fitness)
        return bool(adopted.value)

    # ---- batched group step (phase-level API) ----------------------------------
    def run_group(self, group: int, donor=None):
        """One batched GOM step over colour group `group`; donor (n x |G|,
        GroupBatch order) given explicitly or drawn by the engine."""
        d = None if donor is None else np.ascontiguousarray(donor, np.int32)
        stats = _capi.RunStats()
        crit = self.ctx.control.criteria()
        check(lib().gomix_gpu_run_group(self.h, group, _capi.ptr(d), C.byref(crit), C.byref(stats)))
        self._absorb(stats, self.generation())
        return stats

    def forced_improvement(self, flags=None, group_order=None):
        """One parallel-friendly Forced-Improvement pass now (csrc/gom_fi.cu):
        solutions with flags[s] (None: the engine's own trigger) take the
        elitist as donor group by group in group_order (None: a fresh
        permutation), leave after the first group that strictly improved
        them, else become elitist copies."""
        f = None if flags is None else np.ascontiguousarray(np.asarray(flags) != 0, np.uint8)
        if f is not None and f.shape != (self.n,):
            raise ValueError("forced_improvement: flags must have one entry per solution")
        o = None if group_order is None else np.ascontiguousarray(group_order, np.uint32)
        stats = _capi.RunStats()
        crit = self.ctx.control.criteria()
        check(lib().gomix_gpu_forced_improvement(self.h, _capi.ptr(f), _capi.ptr(o), C.byref(crit), C.byref(stats)))
        self._absorb(stats, self.generation())
        return stats

    def read_batch(self, group: int):
        G = int(self.problem.group_offset[group + 1] - self.problem.group_offset[group])
        d = np.zeros((self.n, G), np.int32)
        de = np.zeros((self.n, G), np.float64)
        p = np.zeros((self.n, G), np.uint8)
        a = np.zeros((self.n, G), np.uint8)
        check(lib().gomix_gpu_read_batch(self.h, d.ctypes.data, de.ctypes.data, p.ctypes.data, a.ctypes.data))
        return d, de, p, a

    # ---- introspection -------------------------------------------------------------
    def population(self, genotypes_out: Optional[np.ndarray] = None, fitness_out: Optional[np.ndarray] = None):
        """(genotypes n x l uint8, fitness n float64); optional caller buffers
        (e.g. pinned host memory) are filled in place."""
        g = genotypes_out if genotypes_out is not None else np.zeros((self.n, self.problem.info.num_vertices), np.uint8)
        f = fitness_out if fitness_out is not None else np.zeros(self.n, np.float64)
        assert g.dtype == np.uint8 and g.shape == (self.n, self.problem.info.num_vertices) and g.flags.c_contiguous
        assert f.dtype == np.float64 and f.shape == (self.n,) and f.flags.c_contiguous
        check(lib().gomix_gpu_read_population(self.h, g.ctypes.data, f.ctypes.data))
        return g, f

    def population_packed(self) -> np.ndarray:
        wp = C.c_uint64()
        check(lib().gomix_gpu_read_population_packed(self.h, None, C.byref(wp)))
        out = np.zeros((self.problem.info.num_vertices, wp.value), np.uint32)
        check(lib().gomix_gpu_read_population_packed(self.h, out.ctypes.data, C.byref(wp)))
        return out

    def group_counters(self):
        k = self.problem.num_groups
        s, st, ca = (np.zeros(k, np.uint64) for _ in range(3))
        check(lib().gomix_gpu_group_counters(self.h, s.ctypes.data, st.ctypes.data, ca.ctypes.data))
        return s, st, ca

    def kernel_times(self) -> np.ndarray:
        cnt = C.c_uint64()
        check(lib().gomix_gpu_kernel_times(self.h, None, 0, C.byref(cnt)))
        buf = np.zeros(max(cnt.value, 1), np.float32)
        check(lib().gomix_gpu_kernel_times(self.h, buf.ctypes.data, cnt.value, C.byref(cnt)))
        return buf[:cnt.value]

    def set_timing(self, enable: bool):
        check(lib().gomix_gpu_set_timing(self.h, int(bool(enable))))

    def kernel_name(self) -> str:
        """The GOM kernel this engine's Philox generations launch."""
        return lib().gomix_gpu_engine_kernel_name(self.h).decode()

    def launch_count(self) -> int:
        c = C.c_uint64()
        check(lib().gomix_gpu_launch_count(self.h, C.byref(c)))
        return c.value


def nccl_unique_id() -> bytes:
    """128-byte NCCL unique id (create on one rank, broadcast to the others)."""
    buf = C.create_string_buffer(128)
    check(lib().gomix_gpu_nccl_unique_id(C.cast(buf, C.c_void_p)))
    return buf.raw


def shard_range(population_size: int, world_size: int, rank: int):
    """Members [lo, hi) held by `rank` (gomix_engine_config sharding rule)."""
    if world_size < 1 or population_size % world_size:
        raise ValueError("population size must be divisible by world_size")
    per = population_size // world_size
    return rank * per, (rank + 1) * per


class _ShardView(GpuParallelEngine):
    """Borrowed handle of one shard of a GpuLocalGroup (read-only helpers)."""

    def __init__(self, problem, handle, n_local, rank, world_size):  # noqa: D107 (no engine creation)
        self.problem, self.h, self.n, self.rank, self.world_size = problem, handle, n_local, rank, world_size
        self.n_global = n_local * world_size

    def __del__(self):
        pass


class GpuLocalGroup:
    """A population sharded over `world_size` engines in this process (one per
    device in `problems`, or several on one device), driven in lock step; the
    per-group exchange is device-to-device copies.  Same arithmetic as one
    process per GPU over NCCL, and equal to a single-engine Philox run."""

    def __init__(self, problems, population_size: int, seed: int = 1, world_size: Optional[int] = None,
                 ctx: Optional[RunContext] = None, transport: str = "copy"):
        """transport "copy": device-to-device copies between the launches;
        "peer": the GOM kernels exchange over peer memory (gom_peer.cuh)."""
        if isinstance(problems, GpuProblem):
            problems = [problems] * int(world_size or 1)
        self.problems = list(problems)
        self.world_size = len(self.problems)
        self.problem = self.problems[0]
        self.n_global = int(population_size)
        shard_range(self.n_global, self.world_size, 0)
        self.ctx = ctx if ctx is not None else RunContext(TerminationConfig(), self.problem.comparator(),
                                                          self.problem.info.num_edges)
        arr = (C.c_void_p * self.world_size)(*[p.h for p in self.problems])
        flags = _capi.FLAG_PEER_TRANSPORT if transport == "peer" else 0
        cfg = _capi.EngineConfig(self.n_global, seed, _capi.MODE_PHILOX, flags, 1, 0, self.world_size, None)
        h = C.c_void_p()
        check(lib().gomix_gpu_local_group_create(C.cast(arr, C.c_void_p), C.byref(cfg), C.byref(h)))
        self.h = h
        self._destroy = lib().gomix_gpu_local_group_destroy
        self.shards = []
        for r in range(self.world_size):
            eh = C.c_void_p()
            check(lib().gomix_gpu_local_group_engine(self.h, r, C.byref(eh)))
            self.shards.append(_ShardView(self.problems[r], eh, self.n_global // self.world_size, r,
                                          self.world_size))
        stats = _capi.RunStats()
        crit = self.ctx.control.criteria()
        check(lib().gomix_gpu_local_group_init_population(self.h, C.byref(crit), C.byref(stats)))
        self.shards[0].ctx = self.ctx
        self.shards[0].pop_id = 1
        self.shards[0]._absorb(stats, 0)

    def __del__(self):
        if getattr(self, "h", None):
            self._destroy(self.h)
            self.h = None

    def run_generation(self):
        ctl = self.ctx.control
        if ctl.stop_requested():
            return
        mg = ctl.cfg.max_generations
        if mg is not None and self.generation() >= mg:  # engine_parallel.hpp:284-289
            ctl.request_stop("generation-limit")
            return
        gen = self.generation()
        stats = _capi.RunStats()
        crit = ctl.criteria()
        check(lib().gomix_gpu_local_group_run_generation(self.h, C.byref(crit), C.byref(stats)))
        self.shards[0]._absorb(stats, gen)
        if not stats.stopped:  # wall clock + trace boundary row, like GpuParallelEngine
            self.ctx.report_boundary(self.shards[0]._elitist_fitness, self.generation(), 1)

    def generation(self) -> int:
        return self.shards[0].generation()

    def population(self):
        parts = [s.population() for s in self.shards]
        return np.concatenate([p[0] for p in parts]), np.concatenate([p[1] for p in parts])

    def elitist(self):
        g = np.zeros(self.problem.info.num_vertices, np.uint8)
        f = C.c_double()
        check(lib().gomix_gpu_local_group_read_elitist(self.h, g.ctypes.data, C.byref(f)))
        return g, f.value

    @property
    def elitist_fitness(self):
        return self.shards[0].elitist_fitness

    def group_counters(self):
        return self.shards[0].group_counters()


def gpu_color(instance: MaxCutInstance, fos: Fos, device: int = 0):
    """GPU Welsh-Powell colouring: (colour per set, k, LMIG edge count)."""
    col = np.zeros(fos.num_sets, np.int32)
    k, e = C.c_uint64(), C.c_uint64()
    check(lib().gomix_gpu_color(C.byref(instance._struct()), C.byref(fos._struct()), device,
                                col.ctypes.data, C.byref(k), C.byref(e)))
    return col, k.value, e.value
