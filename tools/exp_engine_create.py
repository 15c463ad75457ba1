"""Engine construction + first generations wall time (IMS populations are
created during a run, inside its clock)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_08680_b200 as G  # noqa: E402

inst = G.generate_torus(316, 316, ("int", 1, 10), 1)
P = G.GpuProblem(inst, G.univariate_fos(inst.num_vertices))
for n in (16, 16, 128, 1024):
    t0 = time.perf_counter()
    E = G.GpuParallelEngine(P, n, 3, mode="philox")
    t1 = time.perf_counter()
    ts = []
    for _ in range(6):
        a = time.perf_counter()
        E.run_generation()
        ts.append(round(1e3 * (time.perf_counter() - a), 3))
    print(n, "create ms", round(1e3 * (t1 - t0), 2), "generations ms", ts, flush=True)
    del E
