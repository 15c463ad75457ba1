#!/bin/bash
# ncu captures of the dominant kernel (run under gpurun on ONE GPU).
#   tools/profile.sh <tag> <config> [gens] [population]
# -> gpurun_out/<tag>_launches.csv  (every launch, device time)
#    gpurun_out/<tag>.ncu-rep       (--set full of 2 gom_group_kernel launches)
set -u
tag=$1; cfg=$2; gens=${3:-6}; pop=${4:-}
extra=""; [ -n "$pop" ] && extra="--population $pop"
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${tag}_launches.csv \
    python tools/prof_driver.py --config $cfg --gens $gens $extra ${PROF_EXTRA:-} > gpurun_out/${tag}_launches.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:gom_ -s ${SKIP:-4} -c 2 \
    -o gpurun_out/${tag} -f python tools/prof_driver.py --config $cfg --gens $gens $extra ${PROF_EXTRA:-} > gpurun_out/${tag}_full.log 2>&1
echo "profile $tag done"
