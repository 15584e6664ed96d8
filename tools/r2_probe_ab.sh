#!/bin/bash
# skew tests + timings + variants + an ncu capture of the C1 probe (GPU box)
mkdir -p gpurun_out
QUICK=1 bash tools/r2_check.sh
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name regex:"k_local_probe" -c 1 -f -o gpurun_out/r2_probe_new python tools/one_step.py 28 28 1.0 32 1 > gpurun_out/ncu_probe.log 2>&1
tail -2 gpurun_out/ncu_probe.log
