"""Timeline of the persistent generation kernel (C2) from the probes build:

    python -m paper_2203_08680_b200.build --probes
    GOMIX_LIB=paper_2203_08680_b200/libgomix_b200_probes.so python tools/prof_gen_timeline.py [gens]

One generation at a time after warm-up; per colour-group slot, when the
first / last caller reached each point (gom_gen.cu gen_mark), in us from
the first CTA's start."""
import ctypes as C
import json
import sys

sys.path.insert(0, ".")
import numpy as np

import paper_2203_08680_b200 as G
from paper_2203_08680_b200._capi import lib

gens = int(sys.argv[1]) if len(sys.argv) > 1 else 3
inst = G.generate_torus(100, 100, ("int", 1, 10), 1)
P = G.GpuProblem(inst, G.neighbourhood_fos(inst))
E = G.GpuParallelEngine(P, 64, 1, mode="philox")
L = lib()
L.gomix_debug_gen_timeline.argtypes = [C.c_void_p]
buf = np.zeros(128, dtype=np.uint64)
names = ["unit start", "unit done", "cta flushed", "barrier passed", "epilogue done"]
for g in range(30 + gens):
    L.gomix_debug_gen_timeline(C.c_void_p(buf.ctypes.data))  # reset
    E.run_generation()
    if g < 30 and g not in (0, 1, 2):
        continue
    L.gomix_debug_gen_timeline(C.c_void_p(buf.ctypes.data))
    t0 = int(buf[0])
    out = {"generation": g + 1, "cta start": [0.0, round((int(buf[1]) - t0) / 1e3, 2)]}
    slots = []
    for s in range(P.num_groups):
        row = {}
        for i, nm in enumerate(names):
            p = 1 + 6 * s + i
            lo, hi = int(buf[2 * p]), int(buf[2 * p + 1])
            if hi:
                row[nm] = [round((lo - t0) / 1e3, 2), round((hi - t0) / 1e3, 2)]
        slots.append(row)
    out["slots"] = slots
    print(json.dumps(out))
