"""Launch timeline of gom_univ_tt_kernel from the probes build:

    python -m paper_2203_08680_b200.build --probes
    GOMIX_LIB=paper_2203_08680_b200/libgomix_b200_probes.so python tools/prof_timeline.py c3

For one colour-group launch (run_group, Philox, after warm-up generations):
when the first / last CTA reached each point, in us from the first CTA's
start (points: gom_univ.cu timeline_mark calls)."""
import ctypes as C
import json
import sys

sys.path.insert(0, ".")
import numpy as np

import paper_2203_08680_b200 as G
from paper_2203_08680_b200._capi import lib

which = sys.argv[1] if len(sys.argv) > 1 else "c3"
shape, n = {"c3": ((1000, 1000), 128), "c5_16": ((316, 316), 16), "c5_1024": ((316, 316), 1024),
            "c5_4096": ((316, 316), 4096)}[which]
inst = G.generate_torus(shape[0], shape[1], ("int", 1, 10), 1)
P = G.GpuProblem(inst, G.univariate_fos(inst.num_vertices))
E = G.GpuParallelEngine(P, n, 1, mode="philox")
for _ in range(30):
    E.run_generation()
buf = (C.c_ulonglong * 32)()
L = lib()
L.gomix_debug_timeline.argtypes = [C.c_void_p]
names = ["cta start", "prologue done", "warp 0 batches done", "cta flushed", "epilogue start", "epilogue end",
         "all warps' batches done"]
rows = []
for rep in range(3):
    for gi in range(P.num_groups):
        L.gomix_debug_timeline(C.cast(buf, C.c_void_p))  # reset
        E.run_group(gi)
        L.gomix_debug_timeline(C.cast(buf, C.c_void_p))
        v = np.array(buf[:14], dtype=np.float64)
        t0 = v[0]
        row = {"group": gi}
        for i, nm in enumerate(names):
            lo, hi = buf[2 * i], buf[2 * i + 1]
            if hi == 0:
                continue
            row[nm] = [round((lo - t0) / 1e3, 2), round((hi - t0) / 1e3, 2)]
        rows.append(row)
        print(json.dumps(row))
