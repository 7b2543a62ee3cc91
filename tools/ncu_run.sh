#!/bin/bash
# ncu evidence for one bench configuration (run under gpurun on ONE GPU).
#   tools/ncu_run.sh <tag> <bench args...>
# 1) plain run (must exit 0), 2) launch list (gpu__time_duration per launch),
# 3) --set full capture of the pack kernel and the push kernel.
set -u
tag=$1; shift
CMD="python bench.py $*"
mkdir -p gpurun_out
$CMD > gpurun_out/${tag}_plain.log 2>&1 || { echo "plain run failed"; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"pack|push|verify" -c 400 --csv --log-file gpurun_out/${tag}_launches.csv $CMD > gpurun_out/${tag}_ncu_launches.log 2>&1
echo launches=$?
ncu --set full --clock-control none --import-source on -k regex:pack_kernel -s 4 -c 2 -o gpurun_out/${tag}_pack $CMD > gpurun_out/${tag}_ncu_pack.log 2>&1
echo pack=$?
ncu --set full --clock-control none --import-source on -k regex:push_kernel -c 1 -o gpurun_out/${tag}_push $CMD > gpurun_out/${tag}_ncu_push.log 2>&1
echo push=$?
