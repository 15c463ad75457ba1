# The round's GPU evidence in one gpurun call (outputs in gpurun_out/):
#   gpurun --timeout 3600 -- 'bash tools/gpu_validate.sh'
# GPU tests, smoke, the bench lines (C3 default, C2), the reference arm,
# sweeps (C4, C5), the ncu launch list of the bench command (GOM kernels) and
# one `ncu --set full` capture of the C3 truth-table kernel.
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/gputest.txt 2>&1
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.txt 2>&1
timeout 900 python bench.py > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
timeout 900 python bench.py --config c2 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 1200 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_reference_c3.json 2> gpurun_out/bench_reference_c3.err
timeout 900 python tools/sweep.py --c4 --c5 --out-dir gpurun_out > gpurun_out/sweeps.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"gom_|begin_generation|count_ones|presence" \
  -c 300 --csv --log-file gpurun_out/launches_bench_c3.csv \
  python bench.py --steps 20 --warmup 3 --ttt-seconds 0 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:gom_univ_tt_kernel -s 20 -c 1 \
  -o gpurun_out/ncu_c3_tt python bench.py --steps 5 --warmup 3 --ttt-seconds 0 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:gom_generation_kernel -s 10 -c 1 \
  -o gpurun_out/ncu_c2_gen python bench.py --config c2 --steps 5 --warmup 3 --ttt-seconds 0 --no-cpu-baseline > /dev/null 2>&1
