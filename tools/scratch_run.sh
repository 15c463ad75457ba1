cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
L=paper_2203_08680_b200
timeout 900 python -m pytest tests/test_gen_kernel.py tests/test_gpu_parity.py tests/test_configs.py -m gpu -x -q > gpurun_out/g2_tests.log 2>&1; echo tests=$? >> gpurun_out/g2_tests.log
timeout 900 python tools/ab.py --config c2 --rounds 4 --gens 300 flat "two:GOMIX_LIB=$L/libgomix_b200_two.so" > gpurun_out/g2_ab.log 2>&1
