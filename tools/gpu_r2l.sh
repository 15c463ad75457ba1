cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_peer.py tests/test_sharding.py -q --timeout 900 -p no:cacheprovider > gpurun_out/r2l_peer.txt 2>&1
GOMIX_BENCH_ONE_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 2 --steps 10 --warmup 3 --ttt-seconds 10 --e2e-steps 5 > gpurun_out/r2l_bench2.json 2> gpurun_out/r2l_bench2.err
echo "rc=$?" >> gpurun_out/r2l_bench2.err
