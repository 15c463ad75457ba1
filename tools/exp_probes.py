import ctypes as C, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_08680_b200 as G
from paper_2203_08680_b200 import _capi
L = _capi.lib()
L.gomix_debug_probes.argtypes = [C.c_void_p, C.c_int32]
L.gomix_debug_set_flags.argtypes = [C.c_uint32]
inst = G.generate_torus(100, 100, ("int", 1, 10), 1)
P = G.GpuProblem(inst, G.neighbourhood_fos(inst))
for per_group in (False, True):
    E = G.GpuParallelEngine(P, 64, 1, mode="philox", per_group_kernels=per_group)
    for _ in range(20):
        E.run_generation_async()
    E.synchronize()
    buf = np.zeros(64, np.uint64)
    L.gomix_debug_probes(buf.ctypes.data, 1)
    L.gomix_debug_set_flags(32)
    E.run_generation_async(); E.synchronize()
    L.gomix_debug_probes(buf.ctypes.data, 1)
    L.gomix_debug_set_flags(0)
    t0 = buf[0]
    print("per_group" if per_group else "persistent", [(i, int(buf[i] - t0) if buf[i] else None) for i in range(48) if buf[i]])

# per-CTA barrier arrival (slot 0) of the persistent kernel
L.gomix_debug_cta_probes.argtypes = [C.c_void_p]
E = G.GpuParallelEngine(P, 64, 1, mode="philox")
for _ in range(10):
    E.run_generation_async()
E.synchronize()
L.gomix_debug_set_flags(32)
E.run_generation_async(); E.synchronize()
L.gomix_debug_set_flags(0)
cp = np.zeros(8192, np.uint64)
L.gomix_debug_cta_probes(cp.ctypes.data)
t = cp[0::2][:1250].astype(np.int64); sm = cp[1::2][:1250].astype(np.int64)
t = t - t.min()
print("arrival ns: min/median/p90/max", np.percentile(t, [0, 50, 90, 100]))
cnt = np.bincount(sm, minlength=148)
print("CTAs per SM: min/max", cnt.min(), cnt.max(), "hist", np.bincount(cnt))
late = np.argsort(t)[-10:]
print("latest CTAs", late.tolist(), "their SMs", sm[late].tolist(), "load", cnt[sm[late]].tolist())
per_sm_max = np.zeros(148); np.maximum.at(per_sm_max, sm, t)
print("corr(load, SM finish)", np.corrcoef(cnt[cnt > 0], per_sm_max[cnt > 0])[0, 1])
