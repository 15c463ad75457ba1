"""The production (Philox) donor draw has the reference's law: for every
(solution, set) pair the donor is uniform over the members that differ from
the solution on the set — what select_donor's lazy Fisher-Yates scan returns
(engine_serial.hpp:30-46) — and there is none when nobody differs.

Counter-based draws depend on (seed, solution, set, generation), so the same
group step repeated over many seeds on one fixed population samples the law.
"""
import numpy as np
import pytest

import paper_2203_08680_b200 as G

pytestmark = pytest.mark.gpu


def test_philox_donor_is_uniform_over_differing_members():
    inst = G.generate_torus(6, 6, ("int", 1, 5), 3)
    fos = G.neighbourhood_fos(inst)
    P = G.GpuProblem(inst, fos)
    n = 40
    rs = np.random.RandomState(0)
    g0 = (rs.random_sample((n, inst.num_vertices)) < 0.5).astype(np.uint8)
    # make some members agree on the first sets so "same pattern" pools are exercised
    sets0 = [fos.set(int(s)) for s in P.groups[0]]
    g0[1:12][:, sets0[0]] = g0[0, sets0[0]]
    seeds = 1200
    counts = {}
    for seed in range(1, seeds + 1):
        E = G.GpuParallelEngine(P, n, seed, mode="philox", record_batch=True, genotypes=g0)
        E.run_group(0)
        dn, _, pr, _ = E.read_batch(0)
        for s in (0, 5, 20):
            for p in (0, 1, 2):
                counts.setdefault((s, p), []).append(int(dn[s, p]))
    for (s, p), ds in counts.items():
        F = sets0[p]
        differ = np.flatnonzero((g0[:, F] != g0[s, F]).any(axis=1))
        ds = np.array(ds)
        if len(differ) == 0:
            assert (ds == -1).all()
            continue
        assert np.isin(ds, differ).all()
        k = len(differ)
        obs = np.array([(ds == d).sum() for d in differ], float)
        exp = seeds / k
        chi2 = ((obs - exp) ** 2 / exp).sum()
        # chi-square with k-1 dof: mean k-1, sd sqrt(2(k-1)); 6 sd is far out
        assert chi2 < (k - 1) + 6 * np.sqrt(2 * (k - 1)), (s, p, k, chi2)
