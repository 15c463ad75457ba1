"""%globaltimer probes of one truth-table univariate launch (CTA 0: start,
prologue done, batch loop done, flush done; last CTA: epilogue start / end)."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_08680_b200 as G  # noqa: E402
from paper_2203_08680_b200 import _capi  # noqa: E402

L = _capi.lib()
L.gomix_debug_probes.argtypes = [C.c_void_p, C.c_int32]
L.gomix_debug_set_flags.argtypes = [C.c_uint32]
for w, h in ((1000, 1000), (250, 100)):
    inst = G.generate_torus(w, h, ("int", 1, 10), 1)
    P = G.GpuProblem(inst, G.univariate_fos(inst.num_vertices))
    E = G.GpuParallelEngine(P, 128, 1, mode="philox")
    for _ in range(40):
        E.run_generation_async()
    E.synchronize()
    E.set_timing(True)  # launch by launch (the CUDA graph bakes the probe flags in)
    for rep in range(3):
        buf = np.zeros(64, np.uint64)
        L.gomix_debug_probes(buf.ctypes.data, 1)
        L.gomix_debug_set_flags(32)
        E.run_generation_async()
        E.synchronize()
        L.gomix_debug_probes(buf.ctypes.data, 1)
        L.gomix_debug_set_flags(0)
        t0 = int(buf[40])
        print(f"{w}x{h}", {i: (int(buf[i]) - t0) for i in range(40, 46) if buf[i]}, flush=True)
