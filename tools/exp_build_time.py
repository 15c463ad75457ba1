import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_08680_b200 as G
G.GpuProblem(G.generate_torus(4, 4, "unit", 1), G.univariate_fos(16))  # context
cases = [("reg", 4), ("reg", 6), ("reg", 12), ("torus", 1000)]
for kind, arg in cases:
    inst = G.generate_regular(100000, arg, ("real",), seed=arg) if kind == "reg" else G.generate_torus(arg, arg, ("int", 1, 10), 1)
    fos = G.univariate_fos(inst.num_vertices)
    ts = []
    for _ in range(3):
        t0 = time.perf_counter(); P = G.GpuProblem(inst, fos); ts.append(round(time.perf_counter() - t0, 4)); del P
        print("---", kind, arg, ts[-1], file=sys.stderr)
