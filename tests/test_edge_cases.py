"""Edge cases of the GPU engine against the oracle restatement (replay mode,
bit-exact) and by properties (Philox mode): edgeless instances, a single
vertex, a population of one, all-zero weights, the largest linkage set (64
variables), ragged populations (n not a multiple of 32) and sets that are
their own colour class."""
import numpy as np
import pytest

import paper_2203_08680_b200 as G
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _oracle(inst, fos, colour, n, seed):
    return O.OracleEngine(inst.num_vertices, inst.edge_u, inst.edge_v, inst.edge_w, fos.set_offset, fos.set_vars,
                          n, seed, colour=colour)


def _replay_equal(inst, fos, n, seed, gens):
    P = G.GpuProblem(inst, fos)
    Oe = _oracle(inst, fos, P.colour(), n, seed)
    E = G.GpuParallelEngine(P, n, seed, mode="replay")
    for gen in range(gens):
        E.run_generation()
        Oe.run_generation()
        g, f = E.population()
        og, of = Oe.population()
        assert (g == og).all(), gen
        assert (f == of).all(), gen
        assert E.elitist_fitness == Oe.elitist()[1]
    assert E.ctx.control.calls == Oe.evaluator_calls
    return E


def _empty(nv):
    z = np.zeros(0, np.uint32)
    return G.MaxCutInstance(nv, z, z.copy(), np.zeros(0, np.float64))


def test_edgeless_instance():
    inst = _empty(40)
    E = _replay_equal(inst, G.univariate_fos(40), 33, 3, 3)
    assert (E.population()[1] == 0).all()
    P = G.GpuProblem(inst, G.univariate_fos(40))
    F = G.GpuParallelEngine(P, 64, 3, mode="philox")
    for _ in range(3):
        F.run_generation()
    assert (F.population()[1] == 0).all()
    assert F.ctx.control.calls == 0  # no edges: no subfunction is ever evaluated


def test_single_vertex_and_population_of_one():
    inst = _empty(1)
    _replay_equal(inst, G.univariate_fos(1), 5, 1, 2)
    t = G.generate_torus(6, 5, ("int", 1, 10), 2)
    E = _replay_equal(t, G.univariate_fos(t.num_vertices), 1, 4, 3)  # no other member: never a donor
    g0 = E.population()[0]
    for fos in (G.univariate_fos(t.num_vertices), G.neighbourhood_fos(t)):
        F = G.GpuParallelEngine(G.GpuProblem(t, fos), 1, 4, mode="philox")
        g = F.population()[0].copy()
        F.run_generation()
        assert (F.population()[0] == g).all()
    assert g0.shape == (1, t.num_vertices)


def test_all_zero_weights_every_move_is_neutral():
    t = G.generate_torus(7, 6, ("int", 0, 0), 1)
    for fos in (G.univariate_fos(t.num_vertices), G.neighbourhood_fos(t)):
        _replay_equal(t, fos, 40, 2, 3)
        P = G.GpuProblem(t, fos)
        a = G.GpuParallelEngine(P, 64, 5, mode="philox")
        b = G.GpuParallelEngine(P, 64, 5, mode="philox", per_group_kernels=True, lane_per_solution=True)
        for _ in range(3):
            a.run_generation()
            b.run_generation()
        assert (a.population()[0] == b.population()[0]).all()
        assert (a.population()[1] == 0).all()


def test_largest_linkage_set_64_variables():
    t = G.generate_torus(12, 12, ("int", -3, 7), 3)
    nv = t.num_vertices
    sets = [list(range(64))] + [[v] for v in range(64, nv)]  # one 64-variable set, the rest singletons
    fos = G.Fos.from_sets(nv, sets)
    _replay_equal(t, fos, 48, 6, 3)
    P = G.GpuProblem(t, fos)
    F = G.GpuParallelEngine(P, 96, 6, mode="philox")
    for _ in range(3):
        F.run_generation()
    g, f = F.population()
    assert (t.cut_values(g) == f).all()


def test_sets_of_65_variables_are_rejected():
    t = G.generate_torus(12, 12, ("int", 1, 3), 3)
    fos = G.Fos.from_sets(t.num_vertices, [list(range(65))] + [[v] for v in range(65, t.num_vertices)])
    from paper_2203_08680_b200._capi import InvalidArgument

    with pytest.raises(InvalidArgument, match="64 variables"):
        G.GpuProblem(t, fos)


@pytest.mark.parametrize("n", [31, 33, 95, 129, 257])
def test_ragged_populations(n):
    t = G.generate_torus(9, 8, ("int", -2, 9), n)
    _replay_equal(t, G.univariate_fos(t.num_vertices), n, 7, 2)
    F = G.GpuParallelEngine(G.GpuProblem(t, G.neighbourhood_fos(t)), n, 7, mode="philox")
    for _ in range(3):
        F.run_generation()
    g, f = F.population()
    assert (t.cut_values(g) == f).all()
