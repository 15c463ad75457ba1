cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/r2w_gputest.txt 2>&1
for i in 1 2; do timeout 600 python bench.py --ttt-seconds 0 --no-cpu-baseline > gpurun_out/r2w_bench$i.json 2> gpurun_out/r2w_bench$i.err; done
