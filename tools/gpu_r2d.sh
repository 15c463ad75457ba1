cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/r2d_bench_c3.json 2> gpurun_out/r2d_bench_c3.err
timeout 600 python bench.py --config c2 --ttt-seconds 30 > gpurun_out/r2d_bench_c2.json 2> gpurun_out/r2d_bench_c2.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r2d_ref_c3.json 2> gpurun_out/r2d_ref_c3.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2d_launches_c3.csv python bench.py --steps 20 --warmup 3 --ttt-seconds 0 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:gom_univ_tt_kernel -s 20 -c 1 -o gpurun_out/r2d_tt_full python bench.py --steps 5 --warmup 3 --ttt-seconds 0 --no-cpu-baseline > gpurun_out/r2d_ncu.log 2>&1
timeout 600 compute-sanitizer --tool initcheck --print-limit 10 python -m pytest tests/test_gen_kernel.py tests/test_univ_sliced.py -q -p no:cacheprovider > gpurun_out/r2d_initcheck.txt 2>&1
