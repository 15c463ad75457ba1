cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out profiles/r02
for occ in 3 4; do
  GOMIX_TT_OCC=$occ timeout 600 python bench.py --ttt-seconds 0 --no-cpu-baseline > gpurun_out/r2f_bench_occ$occ.json 2> gpurun_out/r2f_bench_occ$occ.err
done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gom_group_kernel -s 10 -c 1 -o gpurun_out/r2f_c4_full python tools/prof_c4.py 4 > gpurun_out/r2f_c4_ncu.log 2>&1
for c in c1 c3 c2; do
  timeout 2400 python tools/success_rate.py --config $c --seeds 30 --out profiles/r02/success_$c.json > gpurun_out/r2f_success_$c.log 2>&1
done
