cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for jb in 256 0 4 16; do echo "== GOMIX_JP_BATCHES=$jb"; GOMIX_JP_BATCHES=$jb GOMIX_TRACE_BUILD=1 timeout 300 python tools/prof_build.py 2>&1 | grep -E "colouring|build [0-9]"; done > gpurun_out/r2q_build.txt 2>&1
timeout 600 python bench.py --config c2 --ttt-seconds 0 --no-cpu-baseline > gpurun_out/r2q_bench_c2.json 2> gpurun_out/r2q_bench_c2.err
