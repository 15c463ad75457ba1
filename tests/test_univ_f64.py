"""The float univariate kernel (csrc/gom_univ_f64.cu, BASELINE C4) against the
lane-per-solution group kernel (csrc/gom.cu) on identical Philox runs.

For a univariate FOS the Philox outcome does not depend on the donor draw, and
both kernels take Σnew and Σold left to right over v's edges in ascending edge
id and apply the same comparator, so every accept decision — populations,
elitists, counters, stop decisions — must be bit-identical.  Fitness deltas
are rounded to fixed point before any sum (order-free integer atomics), so
fitness is bit-identical too, and within 1e-9 relative of the recomputed cut
value (north star).
"""
import numpy as np
import pytest

import paper_2203_08680_b200 as G

pytestmark = pytest.mark.gpu


def _same(inst, a, b, exact=False):
    ga, fa = a.population()
    gb, fb = b.population()
    assert (ga == gb).all()
    assert (fa == fb).all()
    if exact:
        assert (inst.cut_values(ga) == fa).all()
    else:
        assert np.allclose(inst.cut_values(ga), fa, rtol=1e-9, atol=0)
    ea, efa = a.elitist()
    eb, efb = b.elitist()
    assert (ea == eb).all() and efa == efb
    for x, y in zip(a.group_counters(), b.group_counters()):
        assert (x == y).all()


@pytest.mark.parametrize("nv,d,n,gens", [
    (20000, 4, 128, 8),   # C4 shape in small
    (20000, 3, 100, 6),   # odd degree, ragged last word
    (10000, 8, 64, 6),    # 2 words
    (6000, 16, 32, 5),    # C4's largest degree, 1 word
    (3000, 6, 20, 6),     # 20 members
])
def test_f64_kernel_equals_group_kernel(nv, d, n, gens):
    inst = G.generate_regular(nv, d, ("real",), seed=d + n)
    P = G.GpuProblem(inst, G.univariate_fos(nv))
    assert not P.exact
    a = G.GpuParallelEngine(P, n, 3, mode="philox")
    b = G.GpuParallelEngine(P, n, 3, mode="philox", lane_per_solution=True)
    assert a.kernel_name() == "gom_univ_f64_kernel"
    assert b.kernel_name() == "gom_group_kernel"
    _same(inst, a, b)
    for _ in range(gens):
        a.run_generation()
        b.run_generation()
        _same(inst, a, b)


def test_f64_kernel_exact_large_integer_weights():
    """Integer weights too large for the int32 paths: exact comparator,
    fitness by exact atomics."""
    inst = G.generate_torus(24, 20, ("int", 1, 10 ** 12), 5)
    P = G.GpuProblem(inst, G.univariate_fos(inst.num_vertices))
    assert P.exact
    a = G.GpuParallelEngine(P, 96, 2, mode="philox")
    b = G.GpuParallelEngine(P, 96, 2, mode="philox", lane_per_solution=True)
    assert a.kernel_name() == "gom_univ_f64_kernel"
    for _ in range(6):
        a.run_generation()
        b.run_generation()
        _same(inst, a, b, exact=True)


def test_f64_kernel_stop_criteria_and_graph_path():
    inst = G.generate_regular(8000, 4, ("real",), seed=7)
    P = G.GpuProblem(inst, G.univariate_fos(8000))
    for crit in (dict(max_evaluations=700.0), dict(target_fitness=float(inst.edge_w.sum()) * 0.78)):
        ca = G.RunContext(G.TerminationConfig(**crit), P.comparator(), inst.num_edges)
        cb = G.RunContext(G.TerminationConfig(**crit), P.comparator(), inst.num_edges)
        a = G.GpuParallelEngine(P, 64, 5, ctx=ca, mode="philox")
        b = G.GpuParallelEngine(P, 64, 5, ctx=cb, mode="philox", lane_per_solution=True)
        for _ in range(200):
            a.run_generation()
            b.run_generation()
            if ca.control.stop_requested():
                break
        assert ca.control.stop_requested() and cb.control.stop_requested()
        assert ca.control.reason == cb.control.reason
        assert ca.control.calls == cb.control.calls
        _same(inst, a, b)
    # queued generations (the CUDA-graph path) agree with synchronous ones
    a = G.GpuParallelEngine(P, 128, 9, mode="philox")
    b = G.GpuParallelEngine(P, 128, 9, mode="philox")
    for _ in range(10):
        a.run_generation_async()
        b.run_generation()
    a.synchronize()
    _same(inst, a, b)


def test_high_degree_falls_back_to_group_kernel():
    inst = G.generate_regular(2000, 40, ("real",), seed=1)
    P = G.GpuProblem(inst, G.univariate_fos(2000))
    E = G.GpuParallelEngine(P, 64, 1, mode="philox")
    assert E.kernel_name() == "gom_group_kernel"
