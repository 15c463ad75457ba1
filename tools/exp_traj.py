import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_08680_b200 as G
inst = G.generate_torus(100, 100, ("int", 1, 10), 1)
P = G.GpuProblem(inst, G.univariate_fos(10000))
for mode in ("replay", "philox"):
    for lps in (False, True):
        for seed in (1, 2, 3):
            E = G.GpuParallelEngine(P, 64, seed, mode=mode, lane_per_solution=lps)
            tr = []
            for _ in range(15):
                E.run_generation()
                tr.append(E.elitist_fitness)
            print(mode, "lps" if lps else "sliced", seed, tr)
