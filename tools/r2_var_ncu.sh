#!/bin/bash
# variants + ncu of the u64 and C=4 probes (GPU box)
mkdir -p gpurun_out
bash tools/variants.sh 2>&1 | tee gpurun_out/variants.txt
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name regex:"k_local_probe" -c 1 -f -o gpurun_out/r2_probe_u64 python tools/one_step.py 28 28 1.0 64 1 > gpurun_out/ncu_u64.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name regex:"k_local_probe" -c 1 -f -o gpurun_out/r2_probe_c4 python tools/one_step.py 28 28 4.0 32 1 > gpurun_out/ncu_c4.log 2>&1
tail -1 gpurun_out/ncu_u64.log gpurun_out/ncu_c4.log
