cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for g in 0 148 64 16 4 1; do echo "== grid $g"; GOMIX_KAHN_GRID=$g GOMIX_TRACE_BUILD=1 timeout 300 python tools/prof_build.py 2>&1 | grep -E "colouring|build [0-9]" | tail -2; done > gpurun_out/r2v_build.txt 2>&1
