"""Pins the oracle restatement (oracle/gomix_oracle.c) before it is trusted as
the checker: against the reference's own known-answer tests and against the
golden fixtures produced by the unmodified reference (tests/golden/)."""
import numpy as np
import pytest

from oracle import oracle as O
from tests import golden_util as GU

RUN_CASES = ["c1_int", "c1_pm5", "torus6_w", "neigh12", "neigh_n40", "bflt10_40x40", "bflt4_8x8",
             "reg4_float", "reg3_float_neigh", "c2_small_gens"]
COLOR_CASES = ["col_torus10_uni", "col_torus10_neigh", "col_torus100_neigh", "col_torus7x5_uni",
               "col_torus40_bflt10", "col_reg8", "col_reg5odd"]


def test_mix64_kat():  # test_rng.cpp:13-18
    assert O.mix64(0) == 16294208416658607535
    assert O.mix64(0x9E3779B97F4A7C15) == 7960286522194355700
    assert O.mix64(1234567) == 6457827717110365317
    assert O.mix64(42) == 13679457532755275413


def test_mt19937_64_kat():  # test_rng.cpp:20-24
    g = O.MT64(5489, stream=False)
    for _ in range(9999):
        g.next_u64()
    assert g.next_u64() == 9981545732273789042


def test_uniform_index_and_permutation_are_deterministic():  # test_rng.cpp:107-117
    a, b = O.MT64(7), O.MT64(7)
    assert list(a.permutation(20)) == list(b.permutation(20))
    assert sorted(O.MT64(8).permutation(50)) == list(range(50))
    draws = [O.MT64(3).uniform_index(6) for _ in range(3)]
    assert len(set(draws)) == 1 and 0 <= draws[0] < 6


def example_instance():  # test_scheduling.cpp:19-25
    eu = np.array([0, 0, 1, 2, 2, 3], np.uint32)
    ev = np.array([1, 2, 2, 3, 4, 4], np.uint32)
    return 5, eu, ev, np.ones(6)


def example_fos():  # test_scheduling.cpp:29-36
    sets = [[0], [1], [2], [3], [4], [0, 2], [3, 4], [0, 1, 2]]
    off = np.cumsum([0] + [len(s) for s in sets]).astype(np.uint64)
    return off, np.concatenate(sets).astype(np.uint32)


def test_worked_example_lmig_and_frozen_welsh_powell():  # test_scheduling.cpp:64-107
    nv, eu, ev, ew = example_instance()
    off, vars_ = example_fos()
    k, colour, lmig_edges = O.color_sets(nv, eu, ev, ew, off, vars_)
    assert lmig_edges == 22
    assert k == 6
    groups = [sorted(np.flatnonzero(colour == c).tolist()) for c in range(k)]
    assert groups == [[2], [5], [7], [0, 3], [1, 4], [6]]


def test_group_plan_kat():  # test_engine_parallel.cpp:40-56
    eu = np.array([0, 0, 1, 2, 2, 3], np.uint32)
    ev = np.array([1, 2, 2, 3, 4, 4], np.uint32)
    off = np.arange(6, dtype=np.uint64)
    vars_ = np.arange(5, dtype=np.uint32)
    colour = np.array([0, 1, 2, 0, 3], np.int32)  # group 0 = sets {0, 3}
    E = O.OracleEngine(5, eu, ev, np.ones(6), off, vars_, 2, 1, colour=colour)
    ids, fpoff, fp = E.group(0)
    assert ids.tolist() == [0, 3]
    assert fp.tolist() == [0, 1, 3, 5]
    assert fpoff.tolist() == [0, 2, 4]


def test_isolated_vertex_batch_kat():
    """test_engine_parallel.cpp:163-202, mirrored: the reference test hands the
    phases an external elitist {1,1,1}; a whole engine's elitist is the first
    best member, here {0,0,0}, so the roles of the two solutions swap."""
    eu, ev = np.array([0], np.uint32), np.array([1], np.uint32)
    off = np.array([0, 1, 2], np.uint64)
    vars_ = np.array([0, 2], np.uint32)  # one group: sets {0} and {2}
    geno = np.array([[0, 0, 0], [1, 1, 1]], np.uint8)
    E = O.OracleEngine(3, eu, ev, np.ones(1), off, vars_, 2, 1, colour=np.zeros(2, np.int32),
                       genotypes=geno)
    assert E.run_generation() is False
    (gi, donor, delta, present, accept), = E.last_batches()
    steps, calls = E.counters()
    assert int(steps[0]) == 4 and int(calls[0]) == 2
    assert delta[0, 1] == 0.0 and delta[1, 1] == 0.0
    g, f = E.population()
    assert g.tolist() == [[1, 0, 0], [0, 1, 0]]  # elitist keeps its zero-delta gene
    assert f.tolist() == [1.0, 1.0]


def test_torus_generator_matches_reference():
    d = GU.load("c1_int")
    nv, eu, ev, ew = O.generate_torus(10, 10, ("int", 1, 10), 1)
    assert nv == int(d["num_vertices"][0])
    assert (eu == d["edge_u"]).all() and (ev == d["edge_v"]).all() and (ew == d["edge_w"]).all()


@pytest.mark.parametrize("name", COLOR_CASES)
def test_welsh_powell_matches_reference(name):
    d = GU.load(name)
    nv, eu, ev, ew = GU.instance(d)
    off, vars_ = GU.fos(d)
    k, colour, lmig_edges = O.color_sets(nv, eu, ev, ew, off, vars_)
    assert lmig_edges == int(d["lmig_edges"][0])
    assert k == len(d["group_off"]) - 1
    assert (colour == GU.colour_from_groups(d)).all()


@pytest.mark.parametrize("name", RUN_CASES)
def test_engine_matches_reference_run(name):
    d = GU.load(name)
    nv, eu, ev, ew = GU.instance(d)
    off, vars_ = GU.fos(d)
    n, seed, gens = int(d["n"][0]), int(d["seed"][0]), int(d["gens"][0])
    E = O.OracleEngine(nv, eu, ev, ew, off, vars_, n, seed, colour=GU.colour_from_groups(d))
    g, f = E.population()
    assert (g.ravel() == d["init_genotypes"]).all()
    assert (f == d["init_fitness"]).all()
    full = "genotypes" in d
    F = d["fitness"].reshape(gens, n)
    donors, deltas, accepts = [], [], []
    for gen in range(gens):
        E.run_generation()
        g, f = E.population()
        if full:
            assert (g == d["genotypes"].reshape(gens, n, nv)[gen]).all(), gen
        from tests.golden.make_golden import pop_hash
        assert pop_hash(g) == d["pop_hash"][gen]
        assert (f == F[gen]).all(), gen
        assert E.elitist()[1] == d["elitist"][gen]
        assert E.evaluator_calls == int(d["calls"][gen])
        for gi, do, de, p, a in E.last_batches():
            donors.append(do.ravel())
            deltas.append(de.ravel())
            accepts.append(a.ravel())
    if full:
        assert (np.concatenate(donors) == d["donor"]).all()
        assert (np.concatenate(deltas) == d["delta"]).all()
        assert (np.concatenate(accepts) == d["accept"]).all()
    s, c = E.counters()
    assert (s == d["counter_steps"]).all() and (c == d["counter_calls"]).all()
    tf, tc, tg = E.trace()
    assert (tf == d["trace_fitness"]).all()
    assert (tg == d["trace_generation"]).all()
