"""Device problem build of C3 (10^6-vertex torus, univariate FOS), per phase
(GOMIX_TRACE_BUILD=1 prints them on stderr), three repetitions."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_08680_b200 as G  # noqa: E402

G.GpuProblem(G.generate_torus(4, 4, "unit", 1), G.univariate_fos(16))  # context + module load
inst = G.generate_torus(1000, 1000, ("int", 1, 10), 1)
fos = G.univariate_fos(inst.num_vertices)
for _ in range(3):
    t0 = time.perf_counter()
    P = G.GpuProblem(inst, fos)
    print("build s", round(time.perf_counter() - t0, 4), flush=True)
    del P
