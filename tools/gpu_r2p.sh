cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2p_launches_c3.csv python bench.py --steps 20 --warmup 3 --ttt-seconds 0 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:gom_univ_tt_kernel -s 20 -c 1 -o gpurun_out/r2p_tt_full python bench.py --steps 5 --warmup 3 --ttt-seconds 0 --no-cpu-baseline > gpurun_out/r2p_ncu_tt.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:gom_generation_kernel -s 10 -c 1 -o gpurun_out/r2p_gen_full python bench.py --config c2 --steps 5 --warmup 3 --ttt-seconds 0 --no-cpu-baseline > gpurun_out/r2p_ncu_gen.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/r2p_launches_c2.csv python bench.py --config c2 --steps 20 --warmup 3 --ttt-seconds 0 --no-cpu-baseline > /dev/null 2>&1
