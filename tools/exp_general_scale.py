"""General-set throughput at scale: 10^6-vertex torus with neighbourhood and
bounded-FLT FOS (the paper's linkage model), device timing."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2203_08680_b200 as G
from tools.sweep import device_rate
for W in (1000,):
    inst = G.generate_torus(W, W, ("int", 1, 10), 1)
    for name, fos in (("neigh", G.neighbourhood_fos(inst)), ("bflt10", G.bounded_flt_fos(inst, 10)),
                      ("bflt4", G.bounded_flt_fos(inst, 4))):
        t0 = time.perf_counter(); P = G.GpuProblem(inst, fos); b = time.perf_counter() - t0
        for n in (64, 128):
            r = device_rate(G, P, n, gens=10, warm=3)
            print(W, name, n, "sets", fos.num_sets, "groups", P.num_groups, "build", round(b, 2), r, flush=True)
