cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
L=paper_2203_08680_b200
timeout 900 python -m pytest tests/test_univ_sliced.py tests/test_replay_full.py tests/test_gpu_parity.py tests/test_sharding.py tests/test_peer.py -m gpu -x -q > gpurun_out/t2_tests.log 2>&1; echo tests=$? >> gpurun_out/t2_tests.log
timeout 900 python tools/ab.py --rounds 4 --gens 300 new "fence:GOMIX_LIB=$L/libgomix_b200_fence.so" > gpurun_out/t2_ab.log 2>&1
timeout 900 python tools/ab.py --flush --rounds 3 --gens 100 new "fence:GOMIX_LIB=$L/libgomix_b200_fence.so" > gpurun_out/t2_ab_flush.log 2>&1
