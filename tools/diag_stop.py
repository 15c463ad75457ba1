import sys; sys.path.insert(0,'/root/repo')
import numpy as np
import paper_2203_08680_b200 as G
inst = G.generate_torus(20, 20, ("int", 1, 10), 3)
P = G.GpuProblem(inst, G.neighbourhood_fos(inst))
for trial in range(40):
    crit = dict(max_evaluations=333.3)
    ca = G.RunContext(G.TerminationConfig(**crit), P.comparator(), inst.num_edges)
    cb = G.RunContext(G.TerminationConfig(**crit), P.comparator(), inst.num_edges)
    a = G.GpuParallelEngine(P, 64, 9, ctx=ca, mode="philox")
    b = G.GpuParallelEngine(P, 64, 9, ctx=cb, mode="philox", per_group_kernels=True)
    bad = None
    for g in range(300):
        a.run_generation(); b.run_generation()
        ga, fa = a.population(); gb, fb = b.population()
        if not (ga == gb).all() or not (fa == fb).all():
            bad = (g, ca.control.stop_requested(), cb.control.stop_requested(), ca.control.calls, cb.control.calls,
                   int((ga != gb).any(axis=1).sum()), (inst.cut_values(ga) == fa).all(), (inst.cut_values(gb) == fb).all())
            break
        if ca.control.stop_requested() or cb.control.stop_requested():
            break
    print(trial, "gens", g, "bad", bad, flush=True)
