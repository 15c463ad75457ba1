"""Diagnose test_generation_kernel_stop_criteria[crit1] (persistent vs
per-group kernels under an evaluation budget): per-generation states of both
engines, saved for comparison between a plain and a compute-sanitizer run."""
import sys
import numpy as np
sys.path.insert(0, ".")
import paper_2203_08680_b200 as G

tag = sys.argv[1]
crit = dict(max_evaluations=float(sys.argv[2])) if len(sys.argv) > 2 and float(sys.argv[2]) > 0 else {}
inst = G.generate_torus(20, 20, ("int", 1, 10), 3)
P = G.GpuProblem(inst, G.neighbourhood_fos(inst))
out = {}
for name, kw in (("gen", {}), ("grp", dict(per_group_kernels=True))):
    ctx = G.RunContext(G.TerminationConfig(**crit), P.comparator(), inst.num_edges)
    E = G.GpuParallelEngine(P, 64, 9, ctx=ctx, mode="philox", **kw)
    pops, fits, calls, gens = [], [], [], []
    for i in range(60):
        E.run_generation()
        g, f = E.population()
        pops.append(np.packbits(g))
        fits.append(f)
        calls.append(ctx.control.calls)
        gens.append(E.generation())
        if ctx.control.stop_requested():
            break
    out[name + "_pop"] = np.array(pops)
    out[name + "_fit"] = np.array(fits)
    out[name + "_calls"] = np.array(calls)
    out[name + "_gen"] = np.array(gens)
    print(tag, name, "gens run", len(pops), "calls", calls[-1], "reason", ctx.control.reason, "kernel", E.kernel_name())
np.savez(f"gpurun_out/stop_{tag}.npz", **out)
a, b = out["gen_pop"], out["grp_pop"]
m = min(len(a), len(b))
diff = [i for i in range(m) if not (a[i] == b[i]).all()]
print(tag, "first differing generation:", diff[:5], "of", m)
