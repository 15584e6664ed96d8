#!/bin/bash
# ncu --set full of one kernel of one bench-workload step: ncu_one.sh NAME KERNEL_REGEX [one_step args...]
name=$1; kern=$2; shift 2
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name regex:"$kern" -c 1 -f -o gpurun_out/$name python tools/one_step.py "$@" > gpurun_out/ncu_$name.log 2>&1
tail -n 2 gpurun_out/ncu_$name.log
