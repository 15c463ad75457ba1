"""Launch timeline of gom_univ_tt_kernel from the probes build:

    python -m paper_2203_08680_b200.build --probes
    GOMIX_LIB=paper_2203_08680_b200/libgomix_b200_probes.so python tools/prof_timeline.py c3 [graph]

direct (default): one colour-group launch at a time (run_group, Philox,
after warm-up generations); times in us from the first CTA's start.
graph: whole generations as queued CUDA graphs (begin kernel + one launch
per group, programmatic dependent launches); times in us from the begin
kernel's start, per launch.  Each point: when the first / last CTA reached
it (gom_univ.cu timeline_mark calls)."""
import ctypes as C
import json
import sys

sys.path.insert(0, ".")
import numpy as np

import paper_2203_08680_b200 as G
from paper_2203_08680_b200._capi import lib

which = sys.argv[1] if len(sys.argv) > 1 else "c3"
mode = sys.argv[2] if len(sys.argv) > 2 else "direct"
shape, n = {"c3": ((1000, 1000), 128), "c5_16": ((316, 316), 16), "c5_1024": ((316, 316), 1024),
            "c5_4096": ((316, 316), 4096), "tiny": ((16, 16), 128), "c3_100": ((100, 100), 128)}[which]
inst = G.generate_torus(shape[0], shape[1], ("int", 1, 10), 1)
P = G.GpuProblem(inst, G.univariate_fos(inst.num_vertices))
E = G.GpuParallelEngine(P, n, 1, mode="philox")
for _ in range(30):
    E.run_generation()
buf = (C.c_ulonglong * 160)()
L = lib()
L.gomix_debug_timeline.argtypes = [C.c_void_p]
names = ["cta start", "prologue done", "warp 0 batches done", "cta flushed", "epilogue start", "epilogue end",
         "all warps' batches done", "dependency wait over", "epilogue committed", "epilogue control block done",
         "scan chunk maxima", "scan done", "prologue loads back"]


def rows_of(t0, r):
    row = {}
    for i, nm in enumerate(names):
        if nm == "-":
            continue
        lo, hi = buf[32 * r + 2 * i], buf[32 * r + 2 * i + 1]
        if hi == 0:
            continue
        row[nm] = [round((lo - t0) / 1e3, 2), round((hi - t0) / 1e3, 2)]
    return row


if mode == "direct":
    for rep in range(3):
        for gi in range(P.num_groups):
            L.gomix_debug_timeline(C.cast(buf, C.c_void_p))  # reset
            E.run_group(gi)
            L.gomix_debug_timeline(C.cast(buf, C.c_void_p))
            row = {"group": gi}
            row.update(rows_of(buf[0], 0))
            print(json.dumps(row))
else:
    for rep in range(5):
        E.run_generation_async()
        E.synchronize()
        L.gomix_debug_timeline(C.cast(buf, C.c_void_p))  # reset
        E.run_generation_async()
        E.synchronize()
        L.gomix_debug_timeline(C.cast(buf, C.c_void_p))
        t0 = buf[128]
        out = {"rep": rep, "begin kernel": [0.0, round((buf[131] - t0) / 1e3, 2)]}
        for r in range(1, 4):
            row = rows_of(t0, r)
            if row:
                out[f"slot {r - 1}"] = row
        print(json.dumps(out))
