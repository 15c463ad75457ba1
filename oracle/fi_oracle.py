"""CPU restatement of the parallel-friendly Forced Improvement pass
(paper_2203_08680_b200/csrc/gom_fi.cu) for small cases.

TEST INFRASTRUCTURE ONLY (imported by tests/, never by the product package).

The reference has no parallel FI (§5.4 names it future work); its
serial forced_improvement (engine_serial.hpp:98-128) is the model.  This
restates it group-wise, exactly as gom_fi.cu documents:
  * flagged solutions walk the colour groups in `group_order`; in a group,
    every flagged solution that is not yet strictly better than at the start
    of the pass takes the elitist (the group-start elitist genotype) as donor
    on every set of the group where it differs — gom_step's partial
    evaluation and acceptance (engine_serial.hpp:58-86): accept if better, or
    equal and the parent (at group start) is not a copy of the elitist;
  * after each group the elitist scan of engine_parallel.hpp:305-310 (first
    strictly better member, chained);
  * flagged solutions never strictly improved become copies of the elitist.
With singleton groups and one flagged solution this IS the reference's
forced_improvement with the set order = group order (pinned by
tests/test_forced_improvement.py against oracle/_ref/ref_driver's fi mode).
"""
from __future__ import annotations

import numpy as np


def footprint(edge_u, edge_v, vars_):
    s = set(int(x) for x in vars_)
    return np.array([i for i in range(len(edge_u)) if int(edge_u[i]) in s or int(edge_v[i]) in s], np.int64)


def fi_pass(edge_u, edge_v, edge_w, set_off, set_vars, groups, group_order, genotypes, fitness, elit_index,
            elit_fitness, flags):
    """One pass.  groups[c] = set ids of colour c; genotypes n x l (uint8),
    fitness n (float64, integer-valued), elit_index = a column equal to the
    elitist.  Returns (genotypes, fitness, elitist column, elitist fitness,
    evaluator calls, steps)."""
    g = np.array(genotypes, np.uint8, copy=True)
    f = np.array(fitness, np.float64, copy=True)
    n = g.shape[0]
    fit0 = f.copy()
    active = np.asarray(flags, bool).copy()
    e_idx, e_fit = int(elit_index), float(elit_fitness)
    e_geno = g[e_idx].copy()
    fps = {}
    calls = steps = 0
    w = np.asarray(edge_w, np.float64)
    eu, ev = np.asarray(edge_u, np.int64), np.asarray(edge_v, np.int64)
    for c in group_order:
        start = g.copy()
        is_elit = [(start[s] == e_geno).all() for s in range(n)]
        for s in range(n):
            if not active[s] or f[s] > fit0[s]:
                continue
            for sid in groups[c]:
                vars_ = set_vars[set_off[sid]:set_off[sid + 1]].astype(np.int64)
                if (start[s, vars_] == e_geno[vars_]).all():
                    continue
                if sid not in fps:
                    fps[sid] = footprint(eu, ev, vars_)
                fp = fps[sid]
                new = start[s].copy()
                new[vars_] = e_geno[vars_]
                old_cut = (start[s, eu[fp]] != start[s, ev[fp]]).astype(np.float64) @ w[fp]
                new_cut = (new[eu[fp]] != new[ev[fp]]).astype(np.float64) @ w[fp]
                delta = new_cut - old_cut
                calls += len(fp)
                steps += 1
                if delta > 0 or (delta == 0 and not is_elit[s]):
                    g[s, vars_] = e_geno[vars_]
                    f[s] += delta
        # elitist scan (engine_parallel.hpp:305-310)
        for s in range(n):
            if f[s] > e_fit:
                e_fit, e_idx = float(f[s]), s
        e_geno = g[e_idx].copy()
    for s in range(n):
        if active[s] and not f[s] > fit0[s]:
            g[s] = e_geno
            f[s] = e_fit
    return g, f, e_idx, e_fit, calls, steps
