#!/bin/bash
# ncu launch list + full capture of the two-step query's kernels (GPU box)
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name regex:"k_local_build_p|k_repart" --launch-skip 1 -c 3 -f -o gpurun_out/r2_twostep python tools/two_step.py 28 > gpurun_out/ncu_twostep.log 2>&1
tail -2 gpurun_out/ncu_twostep.log
