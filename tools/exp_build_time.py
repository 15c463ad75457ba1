import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_08680_b200 as G
G.GpuProblem(G.generate_torus(4, 4, "unit", 1), G.univariate_fos(16))  # context
for W, kind in ((100, "neigh"), (1000, "uni"), (316, "uni")):
    inst = G.generate_torus(W, W, ("int", 1, 10), 1)
    fos = G.univariate_fos(inst.num_vertices) if kind == "uni" else G.neighbourhood_fos(inst)
    ts = []
    for _ in range(3):
        t0 = time.perf_counter(); P = G.GpuProblem(inst, fos); ts.append(round(time.perf_counter() - t0, 4)); del P
        print("---", ts[-1], file=sys.stderr)
    print(W, kind, "build s (1st, 2nd, 3rd)", ts, file=sys.stderr)
