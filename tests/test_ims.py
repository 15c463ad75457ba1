"""Interleaved multistart (ims.hpp:38-101) and whole runs (run.hpp:41-97).

CPU: the IMS schedule (which population runs when, creation order, sizes,
ids, offer / collect order) with stand-in runners.
GPU: replay-mode IMS runs against the unmodified reference's run_parallel
(golden fixtures from oracle/_ref/ref_driver `ims`): identical improvement
trace (fitness and evaluations), best, stop reason, evaluation count,
generations and population count; Philox IMS solving a small torus; the
device-resident best (collect / offer) against the host elitist API.
"""
import numpy as np
import pytest

import paper_2203_08680_b200 as G
from tests import golden_util as GU


class _Ctl:
    def __init__(self):
        self.stop = False

    def stop_requested(self):
        return self.stop


class _Ctx:
    def __init__(self):
        self.control = _Ctl()


class _Runner:
    def __init__(self, log, size, pid):
        self.log, self.size, self.pid, self.gen = log, size, pid, 0
        log.append(("new", pid, size))

    def run_generation(self):
        self.gen += 1
        self.log.append(("gen", self.pid, self.gen))


class _Best:
    def __init__(self, log):
        self.log = log

    def collect(self, r):
        self.log.append(("collect", r.pid))

    def offer(self, r):
        self.log.append(("offer", r.pid))


def _schedule(base, sub, steps, max_pops=0):
    log = []
    ctx = _Ctx()
    drv = G.GpuImsDriver(G.ImsConfig(base, sub, max_pops), lambda n, pid: _Runner(log, n, pid), ctx, _Best(log))
    for _ in range(steps):
        assert drv.step()
    return drv, log


def test_ims_schedule_interleaves_4_to_1():
    drv, log = _schedule(16, 4, 16)
    gens = [(e[1], e[2]) for e in log if e[0] == "gen"]
    # population 1 runs every step, 2 every 4th, 3 every 16th
    assert gens[:5] == [(1, 1), (1, 2), (1, 3), (1, 4), (2, 1)]
    assert gens[-3:] == [(1, 16), (2, 4), (3, 1)]
    assert [e for e in log if e[0] == "new"] == [("new", 1, 16), ("new", 2, 32), ("new", 3, 64)]
    assert drv.gens == [16, 4, 1]
    # a new population is collected right after creation; every generation is
    # preceded by an offer and followed by a collect (ims.hpp:77-80)
    i = log.index(("new", 2, 32))
    assert log[i + 1:i + 5] == [("collect", 2), ("offer", 2), ("gen", 2, 1), ("collect", 2)]


def test_ims_max_populations_and_validation():
    drv, _ = _schedule(8, 2, 64, max_pops=2)
    assert drv.num_populations() == 2 and drv.gens == [64, 32]
    with pytest.raises(ValueError):
        G.GpuImsDriver(G.ImsConfig(0, 4), None, _Ctx(), None)
    with pytest.raises(ValueError):
        G.GpuImsDriver(G.ImsConfig(16, 0), None, _Ctx(), None)


def test_run_gpu_needs_a_termination_criterion():
    with pytest.raises(ValueError):
        G.ims._require_termination(G.TerminationConfig())


# ---------------------------------------------------------------------------
# GPU
# ---------------------------------------------------------------------------
def _term(d):
    t = d["term"].tolist()
    kw = {}
    for k, v in zip(t[0::2], t[1::2]):
        if k == "--max-evals":
            kw["max_evaluations"] = float(v)
        elif k == "--target":
            kw["target_fitness"] = float(v)
    return G.TerminationConfig(**kw)


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["ims_c1", "ims_pm5", "ims_neigh", "ims_target"])
def test_replay_ims_matches_reference_run_parallel(name):
    d = GU.load(name)
    nv, eu, ev, ew = GU.instance(d)
    inst = G.MaxCutInstance(nv, eu, ev, ew)
    off, vars_ = GU.fos(d)
    P = G.GpuProblem(inst, G.Fos(nv, off, vars_))
    assert (P.group_offset == d["group_off"]).all() and (P.group_sets == d["group_sets"]).all()
    sink = G.RecordingSink()
    r = G.run_gpu(P, _term(d), seed=int(d["seed"][0]), use_ims=True,
                  ims=G.ImsConfig(int(d["base"][0]), int(d["sub"][0])), sink=sink, mode="replay")
    assert [x.fitness for x in sink.rows] == d["trace_fitness"].tolist()
    assert [x.evaluations for x in sink.rows] == d["trace_evals"].tolist()
    assert r.best_fitness == d["best"][0]
    assert inst.cut_value(r.best_genotype) == r.best_fitness
    assert r.reason == str(d["reason"][0])
    assert r.evaluations == d["evaluations"][0]
    assert r.generations == int(d["generations"][0])
    assert r.populations == int(d["populations"][0])


@pytest.mark.gpu
def test_philox_ims_reaches_optimum():
    inst = G.generate_torus(8, 8, "unit", 1)
    P = G.GpuProblem(inst, G.univariate_fos(64))
    r = G.run_gpu(P, G.TerminationConfig(target_fitness=128.0, max_evaluations=1e6), seed=5, use_ims=True,
                  ims=G.ImsConfig(4, 4))
    assert r.reason == "target-reached" and r.best_fitness == 128.0
    assert inst.cut_value(r.best_genotype) == 128.0


@pytest.mark.gpu
def test_device_best_collect_and_offer():
    inst = G.generate_torus(20, 20, ("int", 1, 10), 4)
    P = G.GpuProblem(inst, G.univariate_fos(400))
    a = G.GpuParallelEngine(P, 32, 1, mode="philox")
    b = G.GpuParallelEngine(P, 16, 2, mode="philox")
    for _ in range(5):
        a.run_generation()
    best = G.DeviceBest(P)
    assert best.read() == (None, None)
    best.collect(b)
    gb, fb = best.read()
    eb, efb = b.elitist()
    assert fb == efb and (gb == eb).all()
    best.collect(a)
    ga, fa = best.read()
    ea, efa = a.elitist()
    assert efa > efb and fa == efa and (ga == ea).all()
    best.collect(b)  # not better: unchanged
    assert best.read()[1] == fa
    best.offer(b)     # b adopts a's elitist (strictly better)
    eb2, efb2 = b.elitist()
    assert efb2 == fa and (eb2 == ea).all()
    assert not b.offer_elitist(ea, fa)  # host offer of the same: not strictly better
    # the adopted elitist behaves like a host-offered one: b keeps evolving
    # and its fitness never falls below it
    for _ in range(3):
        b.run_generation()
    assert b.elitist_fitness >= fa
    g, f = b.population()
    assert (inst.cut_values(g) == f).all()
