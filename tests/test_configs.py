"""BASELINE configs at full size: C3 / C4 / C5
shapes through the GPU colouring and Philox engine.

* the GPU Welsh-Powell colouring equals the oracle's sequential greedy
  (oracle/gomix_oracle.c, pinned by the reference's fixtures in
  test_oracle.py) on every colouring path the library has: the shared-memory
  dataflow (<= 10^5 sets), Jones-Plassmann rounds (10^6 univariate), and
  Jones-Plassmann followed by the global dataflow (long chains above 10^5);
* C4 (random d-regular, 10^5 vertices, fp64 weights): colour-class count
  k <= d + 1, fitness equal to the cut values within 1e-9 relative;
* C5 (316 x 316 torus): the population-size extremes n = 16 and n = 4096.
"""
import numpy as np
import pytest

import paper_2203_08680_b200 as G
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _instance(kind, size, arg):
    if kind == "torus":
        return G.generate_torus(size, size, ("int", 1, 10), 1)
    return G.generate_regular(size, arg, ("real",), seed=arg)


@pytest.mark.parametrize("kind,size,arg,fos_kind", [
    ("torus", 316, 0, "neigh"),      # 99,856 sets: shared-memory dataflow
    ("regular", 100000, 16, "uni"),  # C4 d = 16: shared-memory dataflow
    ("torus", 1000, 0, "uni"),       # C3: Jones-Plassmann rounds finish it
    ("torus", 400, 0, "neigh"),      # 160,000 sets in one long chain: JP, then global dataflow
])
def test_gpu_colouring_equals_greedy_at_scale(kind, size, arg, fos_kind):
    inst = _instance(kind, size, arg)
    fos = G.univariate_fos(inst.num_vertices) if fos_kind == "uni" else G.neighbourhood_fos(inst)
    P = G.GpuProblem(inst, fos)
    k, colour, lmig = O.color_sets(inst.num_vertices, inst.edge_u, inst.edge_v, inst.edge_w, fos.set_offset,
                                   fos.set_vars)
    assert P.num_groups == k
    assert P.info.lmig_edges == lmig
    assert (P.colour() == colour).all()


@pytest.mark.parametrize("d", [4, 8, 16])
def test_c4_regular_float_philox(d):
    inst = G.generate_regular(100000, d, ("real",), seed=d)
    P = G.GpuProblem(inst, G.univariate_fos(100000))
    assert not P.exact
    assert 2 <= P.num_groups <= d + 1
    E = G.GpuParallelEngine(P, 128, 3, mode="philox")
    prev = E.elitist_fitness
    for _ in range(3):
        E.run_generation()
        assert E.elitist_fitness >= prev
        prev = E.elitist_fitness
    g, f = E.population()
    assert np.allclose(inst.cut_values(g), f, rtol=1e-9, atol=0)
    sets, steps, calls = E.group_counters()
    assert (calls == steps * d).all()  # every footprint of a d-regular vertex has d edges


@pytest.mark.parametrize("n", [16, 4096])
def test_c5_population_extremes(n):
    inst = G.generate_torus(316, 316, ("int", 1, 10), 1)
    P = G.GpuProblem(inst, G.univariate_fos(inst.num_vertices))
    E = G.GpuParallelEngine(P, n, 2, mode="philox")
    for _ in range(2):
        E.run_generation()
    g, f = E.population()
    assert (inst.cut_values(g) == f).all()
    eg, ef = E.elitist()
    assert inst.cut_value(eg) == ef and f.max() <= ef
