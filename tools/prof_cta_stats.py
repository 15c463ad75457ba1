"""Per-CTA finish times of gom_univ_tt_kernel (probes build):

    python -m paper_2203_08680_b200.build --probes
    GOMIX_LIB=paper_2203_08680_b200/libgomix_b200_probes.so python tools/prof_cta_stats.py [c3]
(path counters: a build with -DGOMIX_PROBES -DGOMIX_PROBE_COUNTS, e.g.
python -m paper_2203_08680_b200.build --variant counts -DGOMIX_PROBES -DGOMIX_PROBE_COUNTS)

One queued generation after warm-up; per launch (graph slot): the spread of
the CTAs' batches-done times, batches per CTA, and finish time by SM and
by batch count — is the launch's tail set by slow SMs, by CTAs that took
more batches, or by single slow batches?"""
import ctypes as C
import json
import sys

sys.path.insert(0, ".")
import numpy as np

import paper_2203_08680_b200 as G
from paper_2203_08680_b200._capi import lib

which = sys.argv[1] if len(sys.argv) > 1 else "c3"
shape, n = {"c3": ((1000, 1000), 128), "c5_1024": ((316, 316), 1024), "c5_4096": ((316, 316), 4096)}[which]
inst = G.generate_torus(shape[0], shape[1], ("int", 1, 10), 1)
P = G.GpuProblem(inst, G.univariate_fos(inst.num_vertices))
E = G.GpuParallelEngine(P, n, 1, mode="philox")
for _ in range(30):
    E.run_generation()
L = lib()
L.gomix_debug_cta_stats.argtypes = [C.c_void_p]
buf = np.zeros(4 * 1024 * 4 + 32, dtype=np.uint64)
CNT = ["batches", "words with accepts", "words with strict improvements", "hash: sparse path", "hash: table path",
       "hash: sum of max accepted sets per solution", "batches with accepts", "words with elitist copies",
       "accepted pairs", "sets with accepts (per word)"]


def counters(label):
    c = buf[4 * 1024 * 4:].astype(np.float64)
    b = max(c[0], 1)
    out = {"phase": label, "batches": int(c[0])}
    for i in range(1, 10):
        out[CNT[i] + " per batch"] = round(c[i] / b, 3)
    print(json.dumps(out))


# path counters: a fresh population's first generations, then the steady state
E2 = G.GpuParallelEngine(P, n, 2, mode="philox")
L.gomix_debug_cta_stats.argtypes = [C.c_void_p]
L.gomix_debug_cta_stats(C.c_void_p(buf.ctypes.data))  # reset
for g in range(1, 6):
    E2.run_generation()
    L.gomix_debug_cta_stats(C.c_void_p(buf.ctypes.data))
    counters(f"fresh population, generation {g}")
for rep in range(3):
    buf[:] = 0
    E.run_generation_async()
    E.synchronize()
    L.gomix_debug_cta_stats(C.c_void_p(buf.ctypes.data))
    counters(f"generation {31 + rep} (steady state)")
    clk = buf[4 * 1024 * 4 + 16:].astype(np.int64)
    # the last launch's epilogue CTA: cycles from epilogue start (point 4)
    pts = {4: "epilogue start", 8: "committed", 9: "control block", 10: "chunk maxima", 11: "scan done",
           5: "epilogue end"}
    print(json.dumps({"epilogue cycles": {nm: int(clk[i] - clk[4]) for i, nm in pts.items() if clk[i]}}))
    st = buf[:4 * 1024 * 4].reshape(4, 1024, 4).astype(np.float64)
    for r in (1, 2):
        rows = st[r][st[r][:, 2] > 0]
        if len(rows) == 0:
            continue
        sm, t0, t1, nb = rows[:, 0], rows[:, 1], rows[:, 2], rows[:, 3]
        base = t0.min()
        fin = (t1 - base) / 1e3
        out = {"rep": rep, "slot": r - 1, "ctas": len(rows),
               "finish_us": [round(float(np.percentile(fin, q)), 2) for q in (0, 10, 50, 90, 100)],
               "batches_per_cta": [int(nb.min()), float(round(nb.mean(), 2)), int(nb.max())]}
        # per-SM finish (max over its CTAs) and per-SM batches
        sms = np.unique(sm)
        smfin = np.array([fin[sm == s].max() for s in sms])
        smnb = np.array([nb[sm == s].sum() for s in sms])
        out["sm_finish_us"] = [round(float(np.percentile(smfin, q)), 2) for q in (0, 10, 50, 90, 100)]
        out["sm_batches"] = [int(smnb.min()), float(round(smnb.mean(), 2)), int(smnb.max())]
        out["corr_finish_batches"] = round(float(np.corrcoef(fin, nb)[0, 1]), 3) if nb.std() > 0 else None
        lo = sm < 74
        out["finish_by_half"] = [round(float(fin[lo].mean()), 2), round(float(fin[~lo].mean()), 2)]
        slow = np.argsort(smfin)[-5:]
        out["slowest_sms"] = [[int(sms[i]), round(float(smfin[i]), 2), int(smnb[i])] for i in slow]
        fast = np.argsort(smfin)[:5]
        out["fastest_sms"] = [[int(sms[i]), round(float(smfin[i]), 2), int(smnb[i])] for i in fast]
        print(json.dumps(out))
