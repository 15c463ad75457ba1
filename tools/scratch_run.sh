cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_replay_full.py -q --timeout 600 -p no:cacheprovider > gpurun_out/r2t_tests.txt 2>&1
