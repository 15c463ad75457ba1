cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for c in c4 c3 c2; do timeout 300 python tools/prof_launch_times.py $c; done > gpurun_out/r2i_launch_times.txt 2>&1
GOMIX_TRACE_BUILD=1 timeout 300 python tools/prof_build.py > gpurun_out/r2i_build.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,sm__cycles_active.avg,smsp__inst_executed.sum --clock-control none -k regex:gom_ --csv --log-file gpurun_out/r2i_c4_launches.csv python tools/prof_c4.py 4 > /dev/null 2>&1
