cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_univ_sliced.py tests/test_replay_full.py tests/test_gpu_parity.py tests/test_sharding.py tests/test_peer.py -q --timeout 900 -p no:cacheprovider > gpurun_out/r2n_tests.txt 2>&1
for c in c3 c5_1024 c5_4096; do
  GOMIX_LIB=paper_2203_08680_b200/libgomix_b200_probes.so timeout 300 python tools/prof_timeline.py $c > gpurun_out/r2n_timeline_$c.txt 2>&1
done
timeout 600 python bench.py --ttt-seconds 0 --no-cpu-baseline > gpurun_out/r2n_bench.json 2> gpurun_out/r2n_bench.err
timeout 900 python tools/sweep.py --c5 --no-ref --out-dir gpurun_out/r2n > gpurun_out/r2n_sweep_c5.log 2>&1
