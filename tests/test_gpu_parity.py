"""GPU parity: the CUDA engine (through the C-ABI) against the reference.

* replay mode vs the golden fixtures the unmodified reference produced
  (tests/golden/, made by oracle/_ref/ref_driver): bit-exact populations,
  fitness, elitist, evaluator calls, group counters, traces, and every
  group's donor / delta / present / accept arrays;
* the GPU Welsh-Powell colouring vs the reference's groups;
* larger seeded cases vs the oracle restatement (oracle/liboracle.so);
* Philox (production) mode vs size-independent properties at full size.
Tolerances: integer weights bit-exact; float weights bit-exact in replay
(reference summation order) and within 1e-9 relative otherwise (north star).
"""
import numpy as np
import pytest

import paper_2203_08680_b200 as G
from oracle import oracle as O
from tests import golden_util as GU

pytestmark = pytest.mark.gpu

RUN_CASES = ["c1_int", "c1_pm5", "torus6_w", "neigh12", "neigh_n40", "bflt10_40x40", "bflt4_8x8",
             "reg4_float", "reg3_float_neigh", "c2_small_gens"]
COLOR_CASES = ["col_torus10_uni", "col_torus10_neigh", "col_torus100_neigh", "col_torus7x5_uni",
               "col_torus40_bflt10", "col_reg8", "col_reg5odd"]


def fixture_problem(d, adopt_groups=False):
    nv, eu, ev, ew = GU.instance(d)
    inst = G.MaxCutInstance(nv, eu, ev, ew)
    off, vars_ = GU.fos(d)
    fos = G.Fos(nv, off, vars_)
    colour = GU.colour_from_groups(d) if adopt_groups else None
    return inst, fos, G.GpuProblem(inst, fos, colour=colour)


def assert_groups_equal(P, d):
    goff = d["group_off"]
    assert P.num_groups == len(goff) - 1
    assert (P.group_offset == goff).all()
    assert (P.group_sets == d["group_sets"]).all()


@pytest.mark.parametrize("name", COLOR_CASES)
def test_gpu_colouring_equals_reference_welsh_powell(name):
    d = GU.load(name)
    inst, fos, P = fixture_problem(d)
    assert_groups_equal(P, d)
    assert P.info.lmig_edges == int(d["lmig_edges"][0])


# univariate integer fixtures run the bit-sliced kernels in replay; each is
# also replayed through the other two univariate kernels
UNIV_INT = ["c1_int", "c1_pm5", "torus6_w"]
KERNEL_VARIANTS = {"default": {}, "adder": dict(truth_table=False), "lane": dict(lane_per_solution=True)}


@pytest.mark.parametrize("name,variant", [(c, "default") for c in RUN_CASES] +
                         [(c, v) for c in UNIV_INT for v in ("adder", "lane")])
def test_replay_generations_match_reference(name, variant):
    """ParallelEngine::run_generation replayed: bit-identical per generation."""
    d = GU.load(name)
    inst, fos, P = fixture_problem(d)
    assert_groups_equal(P, d)
    n, seed, gens = int(d["n"][0]), int(d["seed"][0]), int(d["gens"][0])
    sink = G.RecordingSink()
    ctx = G.RunContext(G.TerminationConfig(), P.comparator(), inst.num_edges, sink)
    E = G.GpuParallelEngine(P, n, seed, ctx=ctx, mode="replay", **KERNEL_VARIANTS[variant])
    if name in UNIV_INT:
        assert E.kernel_name() == {"default": "gom_univ_tt_kernel", "adder": "gom_univ_sliced_kernel",
                                   "lane": "gom_group_kernel"}[variant]
    g, f = E.population()
    assert (g.ravel() == d["init_genotypes"]).all()
    assert (f == d["init_fitness"]).all()
    assert E.elitist_fitness == d["init_elitist"][0]
    assert ctx.control.calls == int(d["init_calls"][0])
    nv = inst.num_vertices
    F = d["fitness"].reshape(gens, n)
    for gen in range(gens):
        E.run_generation()
        g, f = E.population()
        if "genotypes" in d:
            assert (g == d["genotypes"].reshape(gens, n, nv)[gen]).all(), gen
        from tests.golden.make_golden import pop_hash
        assert pop_hash(g) == d["pop_hash"][gen], gen
        assert (f == F[gen]).all(), gen
        eg, ef = E.elitist()
        assert ef == d["elitist"][gen]
        # the elitist's fitness is accumulated (init + deltas) like the
        # reference's; with float weights it equals a fresh evaluation only
        # to within rounding
        assert inst.cut_value(eg) == (ef if P.exact else pytest.approx(ef, rel=1e-12))
        assert ctx.control.calls == int(d["calls"][gen])
        assert E.generation() == gen + 1
    if "final_genotypes" in d:
        assert (g.ravel() == d["final_genotypes"]).all()
    sets, steps, calls = E.group_counters()
    assert (steps == d["counter_steps"]).all() and (calls == d["counter_calls"]).all()
    assert [r.fitness for r in sink.rows] == d["trace_fitness"].tolist()
    assert [r.generation for r in sink.rows] == d["trace_generation"].tolist()
    assert [r.evaluations for r in sink.rows] == d["trace_evals"].tolist()


@pytest.mark.parametrize("name", ["c1_int", "c1_pm5", "torus6_w", "neigh12", "neigh_n40", "bflt4_8x8",
                                  "reg4_float", "reg3_float_neigh"])
def test_batched_group_step_matches_reference_batches(name):
    """Phase-level parity: feed each group the reference's own donor array
    (GroupBatch::donor) and compare delta / present / accept exactly."""
    d = GU.load(name)
    inst, fos, P = fixture_problem(d)
    n, seed, gens = int(d["n"][0]), int(d["seed"][0]), int(d["gens"][0])
    E = G.GpuParallelEngine(P, n, seed, mode="replay", record_batch=True,
                            genotypes=d["init_genotypes"].reshape(n, inst.num_vertices))
    k = P.num_groups
    sizes = [len(x) for x in P.groups]
    at = 0
    for slot, gi in enumerate(d["group_order"].tolist()):
        G_ = sizes[gi]
        sl = slice(at, at + n * G_)
        at += n * G_
        donor = d["donor"][sl].reshape(n, G_)
        E.run_group(gi, donor)
        dn, de, pr, ac = E.read_batch(gi)
        assert (dn == donor).all()
        assert (pr == d["present"][sl].reshape(n, G_)).all(), slot
        assert (de == d["delta"][sl].reshape(n, G_)).all(), slot
        assert (ac == d["accept"][sl].reshape(n, G_)).all(), slot
        if slot % k == k - 1:
            gen = slot // k
            g, f = E.population()
            assert (g == d["genotypes"].reshape(gens, n, inst.num_vertices)[gen]).all()
            assert (f == d["fitness"].reshape(gens, n)[gen]).all()


def test_isolated_vertex_batch_kat():
    """test_engine_parallel.cpp:163-202 (mirrored elitist, see test_oracle)."""
    inst = G.MaxCutInstance(3, np.array([0], np.uint32), np.array([1], np.uint32), np.ones(1))
    fos = G.Fos.from_sets(3, [[0], [2]])
    P = G.GpuProblem(inst, fos, colour=np.zeros(2, np.int32))
    E = G.GpuParallelEngine(P, 2, 1, mode="replay", record_batch=True,
                            genotypes=np.array([[0, 0, 0], [1, 1, 1]], np.uint8))
    E.run_generation()
    d, de, p, a = E.read_batch(0)
    sets, steps, calls = E.group_counters()
    assert int(steps[0]) == 4 and int(calls[0]) == 2
    assert de[0, 1] == 0.0 and de[1, 1] == 0.0
    g, f = E.population()
    assert g.tolist() == [[1, 0, 0], [0, 1, 0]]
    assert f.tolist() == [1.0, 1.0]


def _oracle_for(inst, fos, colour, n, seed):
    return O.OracleEngine(inst.num_vertices, inst.edge_u, inst.edge_v, inst.edge_w, fos.set_offset,
                          fos.set_vars, n, seed, colour=colour)


@pytest.mark.parametrize("shape,weights,fos_kind,n,seed,gens", [
    ((16, 12), ("int", -5, 9), "uni", 100, 3, 6),     # n not a multiple of 32
    ((20, 20), ("int", 1, 3), "neigh", 96, 4, 4),
    ((30, 30), ("int", 1, 10), "uni", 256, 5, 3),      # 8 words / lane
    ((12, 10), ("int", 1, 10), "neigh", 300, 6, 2),    # CTA teams (n > 256)
    ((40, 20), ("int", -3, 3), "uni", 1000, 7, 2),
])
def test_replay_vs_oracle_restatement(shape, weights, fos_kind, n, seed, gens):
    inst = G.generate_torus(shape[0], shape[1], weights, seed)
    fos = G.univariate_fos(inst.num_vertices) if fos_kind == "uni" else G.neighbourhood_fos(inst)
    P = G.GpuProblem(inst, fos)
    Oe = _oracle_for(inst, fos, P.colour(), n, seed)
    k_o = Oe.num_groups
    assert k_o == P.num_groups
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


def test_float_regular_graph_vs_oracle():
    inst = G.generate_regular(400, 6, ("real",), seed=9)
    fos = G.univariate_fos(400)
    P = G.GpuProblem(inst, fos)
    assert not P.exact
    Oe = _oracle_for(inst, fos, P.colour(), 64, 2)
    E = G.GpuParallelEngine(P, 64, 2, mode="replay")
    for _ in range(4):
        E.run_generation()
        Oe.run_generation()
    g, f = E.population()
    og, of = Oe.population()
    assert (g == og).all() and (f == of).all()


@pytest.mark.parametrize("crit", [dict(max_evaluations=1000.0), dict(max_evaluations=777.0),
                                  dict(target_fitness=1000.0), dict(max_generations=3)])
def test_stop_criteria_match_oracle(crit):
    inst = G.generate_torus(10, 10, ("int", 1, 10), 1)
    fos = G.univariate_fos(100)
    P = G.GpuProblem(inst, fos)
    Oe = _oracle_for(inst, fos, P.colour(), 32, 1)
    Oe.set_termination(max_evaluations=crit.get("max_evaluations"), target=crit.get("target_fitness"),
                       max_generations=crit.get("max_generations"))
    ctx = G.RunContext(G.TerminationConfig(**crit), P.comparator(), inst.num_edges)
    E = G.GpuParallelEngine(P, 32, 1, ctx=ctx, mode="replay")
    for _ in range(60):
        E.run_generation()
        Oe.run_generation()
        if ctx.control.stop_requested():
            break
    assert ctx.control.stop_requested()
    assert ctx.control.reason == Oe.stop_reason
    assert E.generation() == Oe.generation
    assert ctx.control.calls == Oe.evaluator_calls
    g, f = E.population()
    og, of = Oe.population()
    assert (g == og).all() and (f == of).all()


def test_offer_elitist_matches_oracle():
    inst = G.generate_torus(8, 8, ("int", 1, 9), 2)
    fos = G.univariate_fos(64)
    P = G.GpuProblem(inst, fos)
    Oe = _oracle_for(inst, fos, P.colour(), 24, 4)
    E = G.GpuParallelEngine(P, 24, 4, mode="replay")
    ext = np.array([(i + i // 8) % 2 for i in range(64)], np.uint8)  # the checkerboard optimum
    fe = inst.cut_value(ext)
    for gen in range(6):
        if gen == 2:
            assert E.offer_elitist(ext, fe)
            Oe.offer_elitist(ext, fe)
            assert not E.offer_elitist(ext, fe)
        E.run_generation()
        Oe.run_generation()
        g, f = E.population()
        og, of = Oe.population()
        assert (g == og).all() and (f == of).all(), gen
    eg, ef = E.elitist()
    og, of = Oe.elitist()
    assert ef == of and (eg == og).all()


# ---------------------------------------------------------------------------
# production (Philox) mode: properties that hold at any size
# ---------------------------------------------------------------------------
def _check_consistent(inst, E, cmp_exact=True):
    g, f = E.population()
    cv = inst.cut_values(g)
    if cmp_exact:
        assert (cv == f).all()
    else:
        assert np.allclose(cv, f, rtol=1e-9, atol=0)
    eg, ef = E.elitist()
    assert f.max() <= ef or np.isclose(f.max(), ef, rtol=1e-9)
    assert inst.cut_value(eg) == pytest.approx(ef, rel=1e-12)


@pytest.mark.parametrize("kind,n", [("uni", 32), ("uni", 128), ("neigh", 64), ("neigh", 512), ("uni", 2048)])
def test_philox_group_step_semantics(kind, n):
    """Every executed pair: donor differs on the set, delta equals the cut
    difference, the accept rule holds (engine_parallel.hpp:104-247)."""
    inst = G.generate_torus(24, 20, ("int", -4, 9), 11)
    fos = G.univariate_fos(inst.num_vertices) if kind == "uni" else G.neighbourhood_fos(inst)
    P = G.GpuProblem(inst, fos)
    E = G.GpuParallelEngine(P, n, 5, mode="philox", record_batch=True)
    for rnd in range(3):
        for gi in range(P.num_groups):
            g0, f0 = E.population()
            _, elit_f = E.elitist()
            elit_g = E.elitist()[0]
            E.run_group(gi)
            dn, de, pr, ac = E.read_batch(gi)
            sets = P.groups[gi]
            g1, f1 = E.population()
            sample = sorted(set(range(min(n, 40))) | set(np.random.RandomState(rnd).choice(n, 8).tolist()))
            for p, sid in enumerate(sets.tolist()):
                F = fos.set(sid)
                for s in sample:
                    differs = (g0[:, F] != g0[s, F]).any(axis=1)
                    assert bool(pr[s, p]) == bool(differs.any())
                    if not pr[s, p]:
                        continue
                    if kind != "uni":
                        assert differs[dn[s, p]]
                        cand = g0[s].copy()
                        cand[F] = g0[dn[s, p], F]
                    else:
                        cand = g0[s].copy()
                        cand[F] = 1 - cand[F]
                    delta = inst.cut_value(cand) - f0[s]
                    assert de[s, p] == delta
                    is_elit = (g0[s] == elit_g).all()
                    expect = delta > 0 or (delta == 0 and not is_elit)
                    assert bool(ac[s, p]) == expect
            _check_consistent(inst, E)


def _nbr_tables(inst):
    """Per vertex its (up to 4) neighbours and edge weights, zero-padded."""
    nv = inst.num_vertices
    nb = np.tile(np.arange(nv)[:, None], (1, 4))
    w = np.zeros((nv, 4))
    cnt = np.zeros(nv, int)
    for a, b, x in zip(inst.edge_u.tolist(), inst.edge_v.tolist(), inst.edge_w.tolist()):
        for p, q in ((a, b), (b, a)):
            nb[p, cnt[p]] = q
            w[p, cnt[p]] = x
            cnt[p] += 1
    return nb, w


@pytest.mark.parametrize("shape,weights,n", [((24, 20), ("int", -4, 9), 128), ((30, 16), ("int", 1, 10), 32),
                                             ((20, 20), ("int", -3, 3), 100), ((18, 14), ("int", 0, 2), 64)])
def test_philox_truth_table_group_step_semantics(shape, weights, n):
    """The benchmarked kernel (gom_univ_tt_kernel, no batch recording) pair by
    pair: (s, {v}) is present iff some member holds the other value; its delta
    is the cut difference of flipping v; it is accepted iff delta > 0 or
    (delta == 0 and s is not the group-start elitist) (engine_parallel.hpp:
    104-247); accepted pairs flip, fitness += sum of accepted deltas."""
    inst = G.generate_torus(shape[0], shape[1], weights, 11)
    P = G.GpuProblem(inst, G.univariate_fos(inst.num_vertices))
    E = G.GpuParallelEngine(P, n, 5, mode="philox")
    assert E.kernel_name() == "gom_univ_tt_kernel"
    nb, w = _nbr_tables(inst)
    for rnd in range(4):
        for gi in range(P.num_groups):
            g0, f0 = E.population()
            eg, _ = E.elitist()
            E.run_group(gi)
            g1, f1 = E.population()
            vs = P.group_sets[P.group_offset[gi]:P.group_offset[gi + 1]].astype(np.int64)
            x = g0[:, vs].astype(bool)
            present = x.min(axis=0) != x.max(axis=0)
            cut = x[:, :, None] != g0[:, nb[vs]].astype(bool)
            delta = (w[vs][None] * (1 - 2 * cut.astype(np.int64))).sum(axis=2)
            is_elit = (g0 == eg).all(axis=1)
            acc = present[None] & ((delta > 0) | ((delta == 0) & ~is_elit[:, None]))
            assert (g1[:, vs].astype(bool) == (x ^ acc)).all(), (rnd, gi)
            rest = np.ones(inst.num_vertices, bool)
            rest[vs] = False
            assert (g1[:, rest] == g0[:, rest]).all()
            assert (f1 == f0 + (acc * delta).sum(axis=1)).all()
    _check_consistent(inst, E)


@pytest.mark.parametrize("kind,shape,n,gens", [("uni", (1000, 1000), 128, 3), ("neigh", (100, 100), 64, 10),
                                               ("uni", (316, 316), 1024, 2)])
def test_philox_full_size_consistency(kind, shape, n, gens):
    """C3 / C2 / C5-size runs: fitness always equals the cut value of the
    genotype (a checksum over every solution), elitist monotone."""
    inst = G.generate_torus(shape[0], shape[1], ("int", 1, 10), 1)
    fos = G.univariate_fos(inst.num_vertices) if kind == "uni" else G.neighbourhood_fos(inst)
    P = G.GpuProblem(inst, fos)
    E = G.GpuParallelEngine(P, n, 1, mode="philox")
    prev = E.elitist_fitness
    for _ in range(gens):
        E.run_generation()
        assert E.elitist_fitness >= prev
        prev = E.elitist_fitness
    _check_consistent(inst, E)
    sets, steps, calls = E.group_counters()
    assert steps.sum() > 0 and (calls >= steps).all()


def test_philox_float_weights_within_tolerance():
    inst = G.generate_regular(20000, 8, ("real",), seed=4)
    P = G.GpuProblem(inst, G.univariate_fos(20000))
    E = G.GpuParallelEngine(P, 128, 3, mode="philox")
    for _ in range(5):
        E.run_generation()
    _check_consistent(inst, E, cmp_exact=False)


def test_philox_solves_small_torus():
    """test_engine_parallel.cpp:243-268: 4x4 unit torus solved to 32."""
    inst = G.generate_torus(4, 4, "unit", 1)
    P = G.GpuProblem(inst, G.univariate_fos(16))
    ctx = G.RunContext(G.TerminationConfig(target_fitness=32.0, max_generations=200), P.comparator(), 32)
    E = G.GpuParallelEngine(P, 24, 8, ctx=ctx, mode="philox")
    while not ctx.control.stop_requested():
        E.run_generation()
    assert ctx.control.reason == "target-reached"
    assert E.elitist_fitness == 32.0
