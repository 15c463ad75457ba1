"""Parallel-friendly Forced Improvement (csrc/gom_fi.cu).

* Pinned to the reference: with singleton colour groups (a complete graph,
  univariate FOS) and one flagged solution, the group-wise pass is the
  reference's forced_improvement (engine_serial.hpp:98-128) with the set order
  = group order — genotype, fitness, evaluator calls and outcome are compared
  with oracle/_ref/ref_driver's fi mode (the unmodified reference), which also
  supplies the order it draws from RngStream(seed).
* Against the CPU restatement (oracle/fi_oracle.py) on multi-set groups with
  many flagged solutions (torus, univariate and neighbourhood FOS).
* The engine flag: fitness stays the cut value, never decreases per solution,
  and runs are deterministic.
"""
import os
import tempfile

import numpy as np
import pytest

import paper_2203_08680_b200 as G
from oracle import fi_oracle as FO
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _complete_graph(m, lo, hi, seed):
    rs = np.random.RandomState(seed)
    u, v = np.triu_indices(m, 1)
    w = rs.randint(lo, hi + 1, len(u)).astype(np.float64)
    return G.MaxCutInstance(m, u.astype(np.uint32), v.astype(np.uint32), w)


def _elitist_column(E):
    g, _ = E.population()
    e, ef = E.elitist()
    idx = [s for s in range(g.shape[0]) if (g[s] == e).all()]
    assert idx, "the elitist is a population column at group boundaries"
    return idx[0], ef


@pytest.mark.skipif(not os.path.exists(O.REF_DRIVER), reason="oracle/_ref not built")
@pytest.mark.parametrize("seed,o_pick", [(1, 0), (2, 1), (3, 2), (4, 3), (5, 4), (6, 5)])
def test_single_solution_equals_reference_forced_improvement(seed, o_pick):
    inst = _complete_graph(14, -6, 9, seed)
    fos = G.univariate_fos(inst.num_vertices)
    P = G.GpuProblem(inst, fos)
    assert P.num_groups == inst.num_vertices  # every set its own group
    E = G.GpuParallelEngine(P, 16, seed, mode="philox")
    for _ in range(2):
        E.run_generation()
    g, f = E.population()
    e_idx, e_fit = _elitist_column(E)
    others = [s for s in range(16) if not (g[s] == g[e_idx]).all()]
    if not others:
        pytest.skip("population converged to the elitist")
    o = others[o_pick % len(others)]
    with tempfile.TemporaryDirectory() as d:
        edges, pop, out = (os.path.join(d, x) for x in ("g.txt", "pop.bin", "fi.bin"))
        G.save_edge_list(edges, inst)
        with open(pop, "wb") as fh:
            fh.write(np.array([16, inst.num_vertices, o, e_idx], np.int64).tobytes())
            fh.write(np.ascontiguousarray(g, np.uint8).tobytes())
        ref = O.run_ref("fi", "--edges", edges, "--fos", "univariate", "--seed", str(100 + seed), "--pop", pop,
                        out=out)
    set_order = ref["set_order"].astype(np.int64)
    group_of = {int(gs[0]): c for c, gs in enumerate(P.groups)}
    order = np.array([group_of[int(sid)] for sid in set_order], np.uint32)
    flags = np.zeros(16, np.uint8)
    flags[o] = 1
    st = E.forced_improvement(flags, order)
    g2, f2 = E.population()
    assert (g2[o] == ref["genotype"]).all()
    assert f2[o] == ref["fitness"][0]
    assert int(st.evaluator_calls) == int(ref["evaluator_calls"][0])
    rest = [s for s in range(16) if s != o]
    assert (g2[rest] == g[rest]).all() and (f2[rest] == f[rest]).all()
    assert (inst.cut_values(g2) == f2).all()


@pytest.mark.parametrize("kind,n,seed", [("uni", 64, 1), ("uni", 100, 2), ("neigh", 64, 3), ("neigh", 32, 4)])
def test_pass_equals_restatement(kind, n, seed):
    inst = G.generate_torus(8, 6, ("int", -4, 9), seed)
    fos = G.univariate_fos(inst.num_vertices) if kind == "uni" else G.neighbourhood_fos(inst)
    P = G.GpuProblem(inst, fos)
    E = G.GpuParallelEngine(P, n, seed, mode="philox")
    for _ in range(3):
        E.run_generation()
    g, f = E.population()
    e_idx, e_fit = _elitist_column(E)
    rs = np.random.RandomState(seed)
    flags = (rs.rand(n) < 0.5).astype(np.uint8)
    order = rs.permutation(P.num_groups).astype(np.uint32)
    calls_before = E.ctx.control.calls
    st = E.forced_improvement(flags, order)
    g2, f2 = E.population()
    rg, rf, _, r_efit, r_calls, r_steps = FO.fi_pass(inst.edge_u, inst.edge_v, inst.edge_w, fos.set_offset,
                                                     fos.set_vars, P.groups, order, g, f, e_idx, e_fit, flags)
    assert (g2 == rg).all()
    assert (f2 == rf).all()
    assert (inst.cut_values(g2) == f2).all()
    assert int(st.evaluator_calls) == r_calls and int(st.steps) == r_steps
    assert E.elitist()[1] == r_efit
    assert E.ctx.control.calls == calls_before + r_calls


def test_engine_flag_runs():
    inst = G.generate_torus(20, 16, ("int", 1, 10), 5)
    for fos in (G.univariate_fos(inst.num_vertices), G.neighbourhood_fos(inst)):
        P = G.GpuProblem(inst, fos)
        a = G.GpuParallelEngine(P, 64, 9, mode="philox", forced_improvement=True)
        b = G.GpuParallelEngine(P, 64, 9, mode="philox", forced_improvement=True)
        prev = a.population()[1]
        for _ in range(12):
            a.run_generation()
            b.run_generation()
            g, f = a.population()
            assert (inst.cut_values(g) == f).all()
            assert (f >= prev).all()  # GOM and FI never make a solution worse
            prev = f
        gb, fb = b.population()
        assert (g == gb).all() and (f == fb).all()
        # FI costs evaluations on top of GOM
        c = G.GpuParallelEngine(P, 64, 9, mode="philox")
        for _ in range(12):
            c.run_generation()
        assert a.ctx.control.calls > c.ctx.control.calls
