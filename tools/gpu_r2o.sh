cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/r2o_gputest.txt 2>&1
timeout 600 python bench.py --ttt-seconds 0 --no-cpu-baseline > gpurun_out/r2o_bench.json 2> gpurun_out/r2o_bench.err
timeout 600 python bench.py --config c2 --ttt-seconds 0 --no-cpu-baseline > gpurun_out/r2o_bench_c2.json 2> gpurun_out/r2o_bench_c2.err
