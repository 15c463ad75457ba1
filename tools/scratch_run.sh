cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python - <<'PY' > gpurun_out/r2s.txt 2>&1
import sys, json
sys.path.insert(0, ".")
sys.path.insert(0, "tools")
import paper_2203_08680_b200 as G
from sweep import device_rate
inst = G.generate_torus(316, 316, ("int", 1, 10), 1)
P = G.GpuProblem(inst, G.univariate_fos(inst.num_vertices))
for n in (256, 384, 512, 512, 640, 768, 1024):
    r = device_rate(G, P, n, gens=20)
    print(json.dumps({k: r[k] for k in ("population", "steps_per_s", "ms_per_generation")}), flush=True)
PY
