cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_univ_f64.py tests/test_gpu_parity.py tests/test_configs.py -q --timeout 600 -p no:cacheprovider > gpurun_out/r2h_tests.txt 2>&1
for occ in 3 2; do GOMIX_F64_OCC=$occ timeout 900 python tools/sweep.py --c4 --out-dir gpurun_out/occ$occ > gpurun_out/r2h_sweep_c4_occ$occ.log 2>&1; done
