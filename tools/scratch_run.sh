cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
L=paper_2203_08680_b200
timeout 900 python -m pytest tests/test_univ_sliced.py tests/test_replay_full.py tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/e1_tests.log 2>&1; echo tests=$? >> gpurun_out/e1_tests.log
timeout 900 python tools/ab.py --rounds 3 --gens 300 early "noearly:GOMIX_TT_EARLY=0" "head:GOMIX_LIB=$L/libgomix_b200_head.so" > gpurun_out/e1_ab.log 2>&1
timeout 900 python tools/ab.py --flush --rounds 3 --gens 100 early "noearly:GOMIX_TT_EARLY=0" "head:GOMIX_LIB=$L/libgomix_b200_head.so" > gpurun_out/e1_ab_flush.log 2>&1
