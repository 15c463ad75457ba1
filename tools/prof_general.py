import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_08680_b200 as G
n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
per_group = len(sys.argv) > 2 and sys.argv[2] == "pg"
inst = G.generate_torus(1000, 1000, ("int", 1, 10), 1)
P = G.GpuProblem(inst, G.neighbourhood_fos(inst))
E = G.GpuParallelEngine(P, n, 1, mode="philox", per_group_kernels=per_group)
for _ in range(3):
    E.run_generation_async()
E.synchronize()
print(E.kernel_name())
