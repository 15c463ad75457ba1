"""Small fixed workload for ncu captures: G Philox generations of a bench
config, or of a C4 d-regular float instance (--regular D)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2203_08680_b200 as G  # noqa: E402
from bench import CONFIGS  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--gens", type=int, default=10)
ap.add_argument("--population", type=int, default=None)
ap.add_argument("--regular", type=int, default=0)
a = ap.parse_args()
if a.regular:
    inst = G.generate_regular(100000, a.regular, ("real",), seed=a.regular)
    fos = G.univariate_fos(inst.num_vertices)
    n = a.population or 128
else:
    cfg = CONFIGS[a.config]
    inst = G.generate_torus(cfg["width"], cfg["height"], cfg["weights"], 1)
    fos = G.univariate_fos(inst.num_vertices) if cfg["fos"] == "uni" else G.neighbourhood_fos(inst)
    n = a.population or cfg["n"]
E = G.GpuParallelEngine(G.GpuProblem(inst, fos), n, 1, mode="philox")
for _ in range(a.gens):
    E.run_generation_async()
E.synchronize()
print("elitist", E.elitist_fitness, "kernel", E.kernel_name())
