"""A few Philox generations of BASELINE C4 (random 4-regular graph, 1e5
vertices, fp64 weights, univariate FOS, n = 128) for ncu captures."""
import sys

sys.path.insert(0, ".")
import paper_2203_08680_b200 as G

d = int(sys.argv[1]) if len(sys.argv) > 1 else 4
inst = G.generate_regular(100000, d, ("real",), seed=d)
P = G.GpuProblem(inst, G.univariate_fos(inst.num_vertices))
E = G.GpuParallelEngine(P, 128, 1, mode="philox")
for _ in range(8):
    E.run_generation()
print(E.kernel_name(), P.num_groups, E.elitist_fitness)
