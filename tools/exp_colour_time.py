"""Device colouring time at the 10^6-set scale: univariate C3 torus and the
neighbourhood FOS of the same torus (GOMIX_TRACE_BUILD=1 prints phases)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_08680_b200 as G  # noqa: E402

G.GpuProblem(G.generate_torus(4, 4, "unit", 1), G.univariate_fos(16))
inst = G.generate_torus(1000, 1000, ("int", 1, 10), 1)
for name, fos in (("uni", G.univariate_fos(inst.num_vertices)), ("neigh", G.neighbourhood_fos(inst))):
    for _ in range(2):
        t0 = time.perf_counter()
        P = G.GpuProblem(inst, fos)
        print(name, "build s", round(time.perf_counter() - t0, 4), "k", P.num_groups, flush=True)
        del P
