"""Per-launch device time of the univariate kernel vs. instance size (fixed
overhead vs. per-set cost), steady state, population 128."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_08680_b200 as G  # noqa: E402

for w, h in ((1000, 1000), (1000, 500), (1000, 250), (500, 250), (250, 100)):
    inst = G.generate_torus(w, h, ("int", 1, 10), 1)
    P = G.GpuProblem(inst, G.univariate_fos(inst.num_vertices))
    for tt in (True, False):
        E = G.GpuParallelEngine(P, 128, 1, mode="philox", truth_table=tt)
        for _ in range(40):
            E.run_generation_async()
        E.synchronize()
        E.set_timing(True)
        E.kernel_times()
        for _ in range(20):
            E.run_generation_async()
        E.synchronize()
        t = E.kernel_times()
        E.set_timing(False)
        print(f"{w}x{h} sets/group={w*h//2} {E.kernel_name():24s} us/launch median {np.median(t)*1e3:.1f} "
              f"min {t.min()*1e3:.1f}", flush=True)
