cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for i in 1 2 3; do timeout 1200 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider 2>&1 | tail -3; done > gpurun_out/r2c_gputest.txt 2>&1
( python tools/debug/stop_race.py plain 333.3
  python tools/debug/stop_race.py plain_nostop 0
  compute-sanitizer --tool memcheck python tools/debug/stop_race.py san 333.3
  compute-sanitizer --tool memcheck python tools/debug/stop_race.py san_nostop 0
) > gpurun_out/r2c_debug.txt 2>&1
for tool in memcheck racecheck synccheck initcheck; do
  echo "== $tool" >> gpurun_out/r2c_sanitizer.txt
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python -m pytest tests/test_gen_kernel.py tests/test_univ_sliced.py -q -p no:cacheprovider -x >> gpurun_out/r2c_sanitizer.txt 2>&1
  echo "rc=$?" >> gpurun_out/r2c_sanitizer.txt
done
