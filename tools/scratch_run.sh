cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
L=paper_2203_08680_b200
timeout 900 python -m pytest tests/test_univ_sliced.py tests/test_replay_full.py tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/s14_tests.log 2>&1; echo tests=$? >> gpurun_out/s14_tests.log
timeout 1500 python tools/ab.py --rounds 2 --gens 300 base "head:GOMIX_LIB=$L/libgomix_b200_head.so" > gpurun_out/ab6.log 2>&1
timeout 1500 python tools/ab.py --config c5 --rounds 2 --gens 100 base "head:GOMIX_LIB=$L/libgomix_b200_head.so" > gpurun_out/ab6_c5.log 2>&1
timeout 1500 python tools/ab.py --config c5 --n 4096 --rounds 2 --gens 50 base "head:GOMIX_LIB=$L/libgomix_b200_head.so" > gpurun_out/ab6_c5_4096.log 2>&1
tail -2 gpurun_out/s14_tests.log; grep round gpurun_out/ab6*.log
