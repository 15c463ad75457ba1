"""Problem-build timing at C3 (GOMIX_TRACE_BUILD=1 prints the phases)."""
import os
import sys
import time

sys.path.insert(0, ".")
os.environ.setdefault("GOMIX_TRACE_BUILD", "1")
import paper_2203_08680_b200 as G

inst = G.generate_torus(1000, 1000, ("int", 1, 10), 1)
fos = G.univariate_fos(inst.num_vertices)
for i in range(4):
    t0 = time.perf_counter()
    P = G.GpuProblem(inst, fos)
    print(f"build {i}: {time.perf_counter() - t0:.4f} s", file=sys.stderr, flush=True)
    del P
