"""The persistent whole-generation kernel (csrc/gom_gen.cu) against one
kernel launch per colour group (csrc/gom.cu) on identical Philox runs.

Both draw the same device group order and the same Philox donors, so
populations, fitness, elitists, group counters, improvement traces and stop
decisions (evaluation budget inside a generation, target) must be
bit-identical; fitness must equal the cut value of every genotype.
"""
import numpy as np
import pytest

import paper_2203_08680_b200 as G

pytestmark = pytest.mark.gpu


def _same(inst, a, b):
    ga, fa = a.population()
    gb, fb = b.population()
    assert (ga == gb).all()
    assert (fa == fb).all()
    assert (inst.cut_values(ga) == fa).all()
    ea, efa = a.elitist()
    eb, efb = b.elitist()
    assert efa == efb and (ea == eb).all()
    assert inst.cut_value(ea) == efa
    for x, y in zip(a.group_counters(), b.group_counters()):
        assert (x == y).all()


@pytest.mark.parametrize("shape,weights,n,gens", [
    ((100, 100), ("int", 1, 10), 64, 6),    # C2
    ((20, 20), ("int", -4, 9), 96, 6),      # signed weights, n % 32 != 0
    ((12, 12), ("int", 1, 10), 20, 8),      # 1 word
    ((16, 10), ("int", 0, 3), 200, 4),      # zero weights, 8 words
    ((9, 7), ("int", 1, 10), 256, 3),       # odd torus, largest supported n
])
def test_generation_kernel_equals_per_group_kernels(shape, weights, n, gens):
    inst = G.generate_torus(shape[0], shape[1], weights, 2)
    P = G.GpuProblem(inst, G.neighbourhood_fos(inst))
    sa, sb = G.RecordingSink(), G.RecordingSink()
    ca = G.RunContext(G.TerminationConfig(), P.comparator(), inst.num_edges, sa)
    cb = G.RunContext(G.TerminationConfig(), P.comparator(), inst.num_edges, sb)
    a = G.GpuParallelEngine(P, n, 5, ctx=ca, mode="philox")
    b = G.GpuParallelEngine(P, n, 5, ctx=cb, mode="philox", per_group_kernels=True)
    assert a.kernel_name() == "gom_generation_kernel"
    assert b.kernel_name() == "gom_group_kernel"
    _same(inst, a, b)
    for _ in range(gens):
        a.run_generation()
        b.run_generation()
        _same(inst, a, b)
    assert [(r.fitness, r.evaluations) for r in sa.rows] == [(r.fitness, r.evaluations) for r in sb.rows]


@pytest.mark.parametrize("crit", [dict(max_evaluations=120.0), dict(max_evaluations=333.3),
                                  dict(target_fitness=2500.0)])
def test_generation_kernel_stop_criteria(crit):
    inst = G.generate_torus(20, 20, ("int", 1, 10), 3)
    P = G.GpuProblem(inst, G.neighbourhood_fos(inst))
    ca = G.RunContext(G.TerminationConfig(**crit), P.comparator(), inst.num_edges)
    cb = G.RunContext(G.TerminationConfig(**crit), P.comparator(), inst.num_edges)
    a = G.GpuParallelEngine(P, 64, 9, ctx=ca, mode="philox")
    b = G.GpuParallelEngine(P, 64, 9, ctx=cb, mode="philox", per_group_kernels=True)
    for _ in range(300):
        a.run_generation()
        b.run_generation()
        if ca.control.stop_requested() or cb.control.stop_requested():
            break
    assert ca.control.stop_requested() and cb.control.stop_requested()
    assert ca.control.reason == cb.control.reason
    assert ca.control.calls == cb.control.calls
    assert a.generation() == b.generation()
    _same(inst, a, b)


def test_generation_kernel_async_and_offer():
    """Queued generations (no host sync) and an offered elitist between them."""
    inst = G.generate_torus(30, 30, ("int", 1, 10), 4)
    P = G.GpuProblem(inst, G.neighbourhood_fos(inst))
    a = G.GpuParallelEngine(P, 64, 1, mode="philox")
    b = G.GpuParallelEngine(P, 64, 1, mode="philox", per_group_kernels=True)
    for _ in range(4):
        a.run_generation_async()
        b.run_generation_async()
    a.synchronize()
    b.synchronize()
    _same(inst, a, b)
    ext = np.array([(i + i // 30) % 2 for i in range(900)], np.uint8)  # checkerboard: cuts every edge
    fe = inst.cut_value(ext)
    assert a.offer_elitist(ext, fe) and b.offer_elitist(ext, fe)
    for _ in range(3):
        a.run_generation()
        b.run_generation()
    _same(inst, a, b)
    assert a.elitist_fitness == fe
