"""The bit-sliced lane-per-set univariate kernel (csrc/gom_univ.cu) against
the lane-per-solution kernel (csrc/gom.cu) on identical Philox runs.

For a univariate FOS the Philox outcome does not depend on the donor draw
(every differing donor holds the flipped bit), so both kernels must produce
bit-identical populations, fitness, elitists, counters and stop decisions —
and fitness must equal the cut value of every genotype (the checksum the
full-size runs use).  Cases cover signed and zero weights, isolated vertices,
populations that are not multiples of 32, every row width (1/2/4 words in one pass, up to
128 words in 4-word passes) and every plane count the kernel instantiates
(4..16).
"""
import numpy as np
import pytest

import paper_2203_08680_b200 as G

pytestmark = pytest.mark.gpu


def _pair(P, n, seed, **kw):
    a = G.GpuParallelEngine(P, n, seed, mode="philox", **kw)
    b = G.GpuParallelEngine(P, n, seed, mode="philox", lane_per_solution=True, **kw)
    return a, b


def _same(inst, a, b):
    ga, fa = a.population()
    gb, fb = b.population()
    assert (ga == gb).all()
    assert (fa == fb).all()
    assert (inst.cut_values(ga) == fa).all()
    ea, efa = a.elitist()
    eb, efb = b.elitist()
    assert efa == efb and (ea == eb).all()
    for x, y in zip(a.group_counters(), b.group_counters()):
        assert (x == y).all()


def _sparse_graph(nv, avg_deg, wlo, whi, seed, isolated=0):
    rs = np.random.RandomState(seed)
    m = nv * avg_deg // 2
    u = rs.randint(0, nv - isolated, m)
    v = rs.randint(0, nv - isolated, m)
    keep = u != v
    a, b = np.minimum(u, v)[keep], np.maximum(u, v)[keep]
    e = np.unique(np.stack([a, b], 1), axis=0)
    w = rs.randint(wlo, whi + 1, len(e)).astype(np.float64)
    return G.MaxCutInstance(nv, e[:, 0].astype(np.uint32), e[:, 1].astype(np.uint32), w)


@pytest.mark.parametrize("shape,weights,n,gens", [
    ((16, 12), ("int", -5, 9), 100, 6),   # signed weights, n % 32 != 0, 4 words
    ((20, 20), ("int", 1, 10), 128, 5),   # C3 shape in small
    ((10, 10), ("int", 1, 10), 32, 8),    # C1 shape, 1 word
    ((14, 9), ("int", -3, 3), 64, 6),     # zero weights, 2 words
    ((9, 7), ("int", 1, 10), 20, 6),      # odd torus (3 colours), 20 members
    ((20, 20), ("int", 1, 10), 256, 4),   # 8 words: two 4-word passes per row
    ((16, 12), ("int", -5, 9), 1000, 3),  # 32 words, last word partial
    ((10, 10), ("int", 1, 10), 4096, 3),  # 128 words, the largest population
])
def test_sliced_equals_lane_per_solution_torus(shape, weights, n, gens):
    inst = G.generate_torus(shape[0], shape[1], weights, 3)
    P = G.GpuProblem(inst, G.univariate_fos(inst.num_vertices))
    a, b = _pair(P, n, 7)
    _same(inst, a, b)
    for _ in range(gens):
        a.run_generation()
        b.run_generation()
        _same(inst, a, b)


@pytest.mark.parametrize("avg_deg,wlo,whi,n", [
    (16, 1, 10, 128),       # A up to ~300: 12 planes
    (6, -1000, 1000, 64),   # 16 planes
    (3, 0, 1, 96),          # 4 planes, many zero weights
    (6, -1000, 1000, 96),   # 16 planes, 4 words: 2-word passes
    (6, -1000, 1000, 256),  # 16 planes, 8 words
    (16, 1, 10, 200),       # 12 planes, 8 words, partial last word
])
def test_sliced_equals_lane_per_solution_random_graphs(avg_deg, wlo, whi, n):
    inst = _sparse_graph(3000, avg_deg, wlo, whi, 5, isolated=40)
    P = G.GpuProblem(inst, G.univariate_fos(inst.num_vertices))
    a, b = _pair(P, n, 9)
    for _ in range(5):
        a.run_generation()
        b.run_generation()
        _same(inst, a, b)


def test_sliced_stop_criteria_match():
    inst = G.generate_torus(30, 30, ("int", 1, 10), 2)
    P = G.GpuProblem(inst, G.univariate_fos(900))
    for crit in (dict(max_evaluations=5000.0), dict(target_fitness=3000.0)):
        ca = G.RunContext(G.TerminationConfig(**crit), P.comparator(), inst.num_edges)
        cb = G.RunContext(G.TerminationConfig(**crit), P.comparator(), inst.num_edges)
        a = G.GpuParallelEngine(P, 64, 3, ctx=ca, mode="philox")
        b = G.GpuParallelEngine(P, 64, 3, ctx=cb, mode="philox", lane_per_solution=True)
        for _ in range(400):
            a.run_generation()
            b.run_generation()
            if ca.control.stop_requested():
                break
        assert ca.control.stop_requested() and cb.control.stop_requested()
        assert ca.control.reason == cb.control.reason
        assert ca.control.calls == cb.control.calls
        assert a.generation() == b.generation()
        _same(inst, a, b)


def test_sliced_full_size_c3():
    """C3 (10^6 vertices, n=128): both kernels agree after two generations and
    fitness is the cut value of every member."""
    inst = G.generate_torus(1000, 1000, ("int", 1, 10), 1)
    P = G.GpuProblem(inst, G.univariate_fos(inst.num_vertices))
    a, b = _pair(P, 128, 1)
    for _ in range(2):
        a.run_generation()
        b.run_generation()
    _same(inst, a, b)


# ---------------------------------------------------------------------------
# truth-table variant (gom_univ_tt_kernel): every variable of degree <= 4
# ---------------------------------------------------------------------------
def _deg4_graph(nv, m, wlo, whi, seed):
    """Random graph with every degree <= 4 (some 0..3), weights in [wlo, whi]."""
    rs = np.random.RandomState(seed)
    deg = np.zeros(nv, np.int64)
    seen, eu, ev = set(), [], []
    for _ in range(m):
        a, b = rs.randint(0, nv, 2)
        a, b = int(min(a, b)), int(max(a, b))
        if a == b or (a, b) in seen or deg[a] >= 4 or deg[b] >= 4:
            continue
        seen.add((a, b))
        deg[a] += 1
        deg[b] += 1
        eu.append(a)
        ev.append(b)
    o = np.lexsort((ev, eu))
    w = rs.randint(wlo, whi + 1, len(eu)).astype(np.float64)
    return G.MaxCutInstance(nv, np.asarray(eu, np.uint32)[o], np.asarray(ev, np.uint32)[o], w)


def _triple(P, n, seed):
    a = G.GpuParallelEngine(P, n, seed, mode="philox")
    b = G.GpuParallelEngine(P, n, seed, mode="philox", truth_table=False)
    c = G.GpuParallelEngine(P, n, seed, mode="philox", lane_per_solution=True)
    assert a.kernel_name() == "gom_univ_tt_kernel"
    assert b.kernel_name() == "gom_univ_sliced_kernel"
    return a, b, c


@pytest.mark.parametrize("inst_kind,n,gens", [
    ("torus_pos", 128, 40),     # long enough for the neutral-oscillation steady state
    ("torus_pm", 100, 25),      # signed weights, partial last word
    ("torus_pm0", 64, 25),      # zero weights, 2 words
    ("torus_c1", 32, 30),       # C1: tiny, clones of the elitist are common
    ("deg4", 128, 25),          # degrees 0..4, padding slots
    ("deg4_big", 96, 20),       # |w| up to 8000: 16 planes
    # n > 128: rows in 4-word chunks, one chunk per CTA, presence from the
    # per-generation row counts
    ("torus_pos", 256, 20),     # 2 chunks
    ("torus_pm", 1000, 12),     # 8 chunks, last one partial (1000 = 7 x 128 + 104)
    ("torus_c1", 4096, 8),      # 32 chunks: the largest population
    ("deg4", 520, 10),          # padding slots, ragged last chunk
    ("deg4_big", 384, 8),       # 16 planes, 3 chunks
])
def test_truth_table_equals_adder_and_lane_per_solution(inst_kind, n, gens):
    inst = {
        "torus_pos": lambda: G.generate_torus(24, 20, ("int", 1, 10), 4),
        "torus_pm": lambda: G.generate_torus(16, 12, ("int", -5, 9), 3),
        "torus_pm0": lambda: G.generate_torus(14, 9, ("int", -3, 3), 3),
        "torus_c1": lambda: G.generate_torus(10, 10, ("int", 1, 10), 1),
        "deg4": lambda: _deg4_graph(2000, 5000, -5, 9, 11),
        "deg4_big": lambda: _deg4_graph(1500, 4000, -8000, 8000, 12),
    }[inst_kind]()
    P = G.GpuProblem(inst, G.univariate_fos(inst.num_vertices))
    a, b, c = _triple(P, n, 5)
    for _ in range(gens):
        for e in (a, b, c):
            e.run_generation()
        _same(inst, a, b)
        _same(inst, a, c)


def test_truth_table_stop_criteria_match():
    inst = G.generate_torus(30, 30, ("int", 1, 10), 2)
    P = G.GpuProblem(inst, G.univariate_fos(900))
    for crit in (dict(max_evaluations=5000.0), dict(target_fitness=3000.0)):
        ca = G.RunContext(G.TerminationConfig(**crit), P.comparator(), inst.num_edges)
        cb = G.RunContext(G.TerminationConfig(**crit), P.comparator(), inst.num_edges)
        a = G.GpuParallelEngine(P, 64, 3, ctx=ca, mode="philox")
        b = G.GpuParallelEngine(P, 64, 3, ctx=cb, mode="philox", truth_table=False)
        for _ in range(400):
            a.run_generation()
            b.run_generation()
            if ca.control.stop_requested():
                break
        assert ca.control.stop_requested() and cb.control.stop_requested()
        assert ca.control.reason == cb.control.reason
        assert ca.control.calls == cb.control.calls
        _same(inst, a, b)


def test_truth_table_full_size_c3():
    """C3 (10^6 vertices, n=128): the truth-table kernel (the bench's) agrees
    with the adder kernel over 30 generations (into the steady state)."""
    inst = G.generate_torus(1000, 1000, ("int", 1, 10), 1)
    P = G.GpuProblem(inst, G.univariate_fos(inst.num_vertices))
    a = G.GpuParallelEngine(P, 128, 1, mode="philox")
    b = G.GpuParallelEngine(P, 128, 1, mode="philox", truth_table=False)
    assert a.kernel_name() == "gom_univ_tt_kernel"
    for _ in range(30):
        a.run_generation_async()
        b.run_generation_async()
    a.synchronize()
    b.synchronize()
    _same(inst, a, b)


def test_truth_table_full_size_c5_large_population():
    """C5 at the top of its sweep (316 x 316 torus, n = 4096: 32 chunks per
    row): the chunked truth-table kernel agrees with the adder kernel."""
    inst = G.generate_torus(316, 316, ("int", 1, 10), 1)
    P = G.GpuProblem(inst, G.univariate_fos(inst.num_vertices))
    a = G.GpuParallelEngine(P, 4096, 1, mode="philox")
    b = G.GpuParallelEngine(P, 4096, 1, mode="philox", truth_table=False)
    assert a.kernel_name() == "gom_univ_tt_kernel" and b.kernel_name() == "gom_univ_sliced_kernel"
    for _ in range(6):
        a.run_generation_async()
        b.run_generation_async()
    a.synchronize()
    b.synchronize()
    _same(inst, a, b)
