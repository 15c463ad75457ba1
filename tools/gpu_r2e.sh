cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_univ_sliced.py tests/test_replay_full.py tests/test_gpu_parity.py -q --timeout 900 -p no:cacheprovider > gpurun_out/r2e_tests.txt 2>&1
for occ in 3 4; do
  GOMIX_TT_OCC=$occ timeout 600 python bench.py --ttt-seconds 0 --no-cpu-baseline > gpurun_out/r2e_bench_occ$occ.json 2> gpurun_out/r2e_bench_occ$occ.err
done
timeout 900 python tools/sweep.py --c5 --no-ref --out-dir gpurun_out > gpurun_out/r2e_sweep.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:gom_univ_tt_kernel -s 20 -c 1 -o gpurun_out/r2e_tt_full python bench.py --steps 5 --warmup 3 --ttt-seconds 0 --no-cpu-baseline > gpurun_out/r2e_ncu.log 2>&1
