import sys, os, time, cProfile, pstats
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_08680_b200 as G
cfgs = {"c3": (1000, "uni"), "c2": (100, "neigh")}
for name in sys.argv[1:] or ["c3"]:
    W, kind = cfgs[name]
    inst = G.generate_torus(W, W, ("int", 1, 10), 1)
    fos = G.univariate_fos(inst.num_vertices) if kind == "uni" else G.neighbourhood_fos(inst)
    t0 = time.perf_counter(); P = G.GpuProblem(inst, fos); print(name, "build", time.perf_counter() - t0)
    G.run_gpu(P, G.TerminationConfig(max_seconds=0.5), seed=9)  # warm
    pr = cProfile.Profile(); pr.enable()
    r = G.run_gpu(P, G.TerminationConfig(max_seconds=2.0), seed=1)
    pr.disable()
    print(name, "pops", r.populations, "gens(pop1)", r.generations, "evals", r.evaluations, "best", r.best_fitness)
    pstats.Stats(pr).sort_stats("tottime").print_stats(12)
