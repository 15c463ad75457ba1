"""Per-launch CUDA-event durations of the GOM kernels of one config
(E.set_timing: launch by launch) next to graph-path generation times."""
import json
import sys

sys.path.insert(0, ".")
import numpy as np
import torch

import paper_2203_08680_b200 as G

which = sys.argv[1] if len(sys.argv) > 1 else "c4"
if which == "c4":
    inst = G.generate_regular(100000, 4, ("real",), seed=4)
    fos = G.univariate_fos(inst.num_vertices)
    n = 128
elif which == "c3":
    inst = G.generate_torus(1000, 1000, ("int", 1, 10), 1)
    fos = G.univariate_fos(inst.num_vertices)
    n = 128
else:
    inst = G.generate_torus(100, 100, ("int", 1, 10), 1)
    fos = G.neighbourhood_fos(inst)
    n = 64
P = G.GpuProblem(inst, fos)
s = torch.cuda.Stream()
E = G.GpuParallelEngine(P, n, 1, mode="philox", stream=s.cuda_stream)
for _ in range(20):
    E.run_generation_async()
E.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(s)
for _ in range(20):
    E.run_generation_async()
e1.record(s)
E.synchronize()
torch.cuda.synchronize()
graph_ms = e0.elapsed_time(e1) / 20
E.set_timing(True)
E.kernel_times()
for _ in range(20):
    E.run_generation_async()
E.synchronize()
kt = E.kernel_times()
print(json.dumps({"config": which, "kernel": E.kernel_name(), "groups": P.num_groups,
                  "graph_ms_per_generation": graph_ms, "launch_ms_mean": float(np.mean(kt)),
                  "launch_ms_min": float(np.min(kt)), "launch_ms_max": float(np.max(kt)),
                  "launches": int(len(kt)), "sum_launch_ms_per_generation": float(np.sum(kt)) / 20}))
