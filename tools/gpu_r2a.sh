cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2a_smi.txt
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/r2a_gputest.txt 2>&1
echo "gputest rc=$?" >> gpurun_out/r2a_gputest.txt
timeout 300 python __graft_entry__.py smoke > gpurun_out/r2a_smoke.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/r2a_smoke.txt
for i in 1 2 3 4 5 6; do GOMIX_ALLOC_CACHE=1 timeout 300 python -m pytest tests/test_gen_kernel.py -q -p no:cacheprovider 2>&1 | tail -2; done > gpurun_out/r2a_flaky.txt 2>&1
for tool in memcheck racecheck synccheck initcheck; do
  echo "== $tool" >> gpurun_out/r2a_sanitizer.txt
  timeout 600 compute-sanitizer --tool $tool --print-limit 20 python -m pytest tests/test_gen_kernel.py -q -p no:cacheprovider -k "stop_criteria" >> gpurun_out/r2a_sanitizer.txt 2>&1
  echo "rc=$?" >> gpurun_out/r2a_sanitizer.txt
done
