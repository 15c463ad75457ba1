cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
( python tools/debug/stop_race.py plain 333.3
  python tools/debug/stop_race.py plain_nostop 0
  compute-sanitizer --tool memcheck python tools/debug/stop_race.py san 333.3
  compute-sanitizer --tool memcheck python tools/debug/stop_race.py san_nostop 0
) > gpurun_out/r2b_debug.txt 2>&1
