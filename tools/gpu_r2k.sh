cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_sharding.py tests/test_capi.py -q --timeout 600 -p no:cacheprovider -x > gpurun_out/r2k_sharding.txt 2>&1
timeout 900 python -m pytest tests/test_peer.py -q --timeout 600 -p no:cacheprovider -x > gpurun_out/r2k_peer.txt 2>&1
