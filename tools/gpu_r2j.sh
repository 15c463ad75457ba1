cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/r2j_gputest.txt 2>&1
timeout 900 python tools/sweep.py --c4 --out-dir gpurun_out/r2j > gpurun_out/r2j_sweep_c4.log 2>&1
timeout 900 python tools/sweep.py --c5 --no-ref --out-dir gpurun_out/r2j > gpurun_out/r2j_sweep_c5.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gom_univ_f64_kernel -s 15 -c 5 -o gpurun_out/r2j_c4_f64 python tools/prof_c4.py 4 > gpurun_out/r2j_c4_ncu.log 2>&1
