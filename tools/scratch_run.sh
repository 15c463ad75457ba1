cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
L=paper_2203_08680_b200
timeout 900 python -m pytest tests/test_univ_sliced.py tests/test_replay_full.py tests/test_gpu_parity.py tests/test_univ_f64.py tests/test_ims.py -m gpu -x -q > gpurun_out/s8_tests.log 2>&1; echo tests=$? >> gpurun_out/s8_tests.log
timeout 1500 python tools/ab.py --rounds 3 --gens 300 base "head:GOMIX_LIB=$L/libgomix_b200_head.so" "graph:GOMIX_GRAPH=1" > gpurun_out/ab2.log 2>&1
tail -3 gpurun_out/s8_tests.log; grep -A3 '"base"\|"head"\|"graph"' gpurun_out/ab2.log | grep -v kernel
