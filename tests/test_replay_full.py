"""Replay parity of the benchmarked bit-sliced univariate kernels against the
unmodified reference at the BASELINE sizes.

The fixtures (tests/golden/c3_full.npz, c5_n16, c5_n1024, c1_long, c3_pm) were
made by `python tests/golden/make_golden.py --light`: the reference's
ParallelEngine (oracle/_ref/ref_driver, compiled from its headers) run for a
few generations, every generation's population hashed (sha256 of
numpy.packbits of the n x l genotype bytes), fitness arrays, elitist,
evaluator calls, group counters and traces kept whole.

In replay mode the engine walks the reference's RngStream on the host
(init bits, `permutation(k)`, every lazy Fisher-Yates donor scan,
engine_serial.hpp:30-46, rng.hpp:21-59) and launches the SAME kernel the
Philox production path launches (gom_univ_tt_kernel; rows above 4 words in
4-word chunks, one per CTA): univariate steps are donor-independent, only
presence and the group order matter.  Integer weights: bit-exact.
"""
import numpy as np
import pytest

import paper_2203_08680_b200 as G
from tests import golden_util as GU
from tests.golden.make_golden import array_hash, packed_hash

pytestmark = pytest.mark.gpu

# fixture -> the kernel its Philox and replay generations launch
EXPECT = {
    "c1_long": "gom_univ_tt_kernel",      # C1: n = 32, one word per row
    "c3_pm": "gom_univ_tt_kernel",        # signed weights, n = 100 (ragged last word)
    "c5_n16": "gom_univ_tt_kernel",       # C5 smallest population
    "c5_n1024": "gom_univ_tt_kernel",     # C5, 32 words per row: 8 chunks of 4 words
    "c3_full": "gom_univ_tt_kernel",      # C3 as benchmarked: 10^6 vertices, n = 128
    # C4: fp64 weights on random d-regular graphs (this repo's generator,
    # handed to the reference as an edge-list file): float replay keeps the
    # reference's summation order, so fitness too is bit for bit
    "c4_d4": "gom_group_kernel",          # 10^5 vertices, d = 4, n = 128
    "c4_d8_small": "gom_group_kernel",    # 2 x 10^4 vertices, d = 8, n = 64
}


def _weights(spec: str):
    if spec == "unit":
        return "unit"
    _, lo, hi = spec.split(":")
    return ("int", int(lo), int(hi))


def light_problem(d):
    w, h = (int(x) for x in d["torus"])
    if w or "regular" not in d:
        inst = G.generate_torus(w, h, _weights(str(d["weights"][0])), int(d["inst_seed"][0]))
    else:
        nv, deg, gseed = (int(x) for x in d["regular"])
        inst = G.generate_regular(nv, deg, ("real",), seed=gseed)
    assert array_hash(inst.edge_u, inst.edge_v, inst.edge_w) == d["edges_hash"][0], "instance generator drifted"
    P = G.GpuProblem(inst, G.univariate_fos(inst.num_vertices))
    assert (P.group_offset == d["group_off"]).all()
    assert array_hash(P.group_sets.astype(np.uint64)) == d["group_sets_hash"][0]
    return inst, P


def run_light(name, **engine_kw):
    d = GU.load(name)
    inst, P = light_problem(d)
    n, seed, gens = int(d["n"][0]), int(d["seed"][0]), int(d["gens"][0])
    sink = G.RecordingSink()
    ctx = G.RunContext(G.TerminationConfig(), P.comparator(), inst.num_edges, sink)
    E = G.GpuParallelEngine(P, n, seed, ctx=ctx, mode="replay", **engine_kw)
    g, f = E.population()
    assert packed_hash(np.packbits(g)) == d["init_hash"][0]
    assert (f == d["init_fitness"]).all()
    assert E.elitist_fitness == d["init_elitist"][0]
    assert ctx.control.calls == int(d["init_calls"][0])
    F = d["fitness"].reshape(gens, n)
    for gen in range(gens):
        E.run_generation()
        g, f = E.population()
        assert packed_hash(np.packbits(g)) == d["pop_hash"][gen], gen
        assert (f == F[gen]).all(), gen
        assert E.elitist_fitness == d["elitist"][gen], gen
        assert ctx.control.calls == int(d["calls"][gen]), gen
        assert E.generation() == gen + 1
    eg, ef = E.elitist()
    # the elitist's fitness is accumulated (init + deltas) like the
    # reference's: with float weights it equals a fresh evaluation only to
    # within rounding
    assert inst.cut_value(eg) == (ef if P.exact else pytest.approx(ef, rel=1e-12))
    _, steps, calls = E.group_counters()
    assert (steps == d["counter_steps"]).all() and (calls == d["counter_calls"]).all()
    assert [r.fitness for r in sink.rows] == d["trace_fitness"].tolist()
    assert [r.generation for r in sink.rows] == d["trace_generation"].tolist()
    assert [r.evaluations for r in sink.rows] == d["trace_evals"].tolist()
    return E


@pytest.mark.parametrize("name", list(EXPECT))
def test_replay_full_size_matches_reference(name):
    E = run_light(name)
    assert E.kernel_name() == EXPECT[name]


@pytest.mark.parametrize("name,variant", [(c, v) for c in ("c1_long", "c3_pm", "c5_n16")
                                          for v in (dict(truth_table=False), dict(lane_per_solution=True))]
                         + [("c5_n1024", dict(truth_table=False))])
def test_replay_full_size_other_kernels(name, variant):
    """The adder kernel (gom_univ_sliced_kernel) and the lane-per-solution
    kernel (gom_group_kernel, donor tape) give the same bit-exact replay."""
    E = run_light(name, **variant)
    assert E.kernel_name() == ("gom_group_kernel" if "lane_per_solution" in variant else "gom_univ_sliced_kernel")
