#!/bin/bash
# skew timings (2^24 then 2^28) + ncu full captures of probe / local build / part2 at C=1 and C=4
mkdir -p gpurun_out
timeout 300 python tools/skew.py 24 > gpurun_out/skew24.jsonl 2> gpurun_out/skew24.err; echo "skew24 rc=$?" >> gpurun_out/skew24.err
timeout 600 python tools/skew.py 28 > gpurun_out/skew28.jsonl 2> gpurun_out/skew28.err; echo "skew28 rc=$?" >> gpurun_out/skew28.err
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name regex:"k_local_probe|k_part2|k_local_build_p" -c 4 -f -o gpurun_out/r2_c1 python tools/one_step.py 28 28 1.0 32 1 > gpurun_out/ncu_c1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name regex:"k_local_probe" -c 1 -f -o gpurun_out/r2_c4 python tools/one_step.py 28 28 4.0 32 1 > gpurun_out/ncu_c4.log 2>&1
tail -2 gpurun_out/ncu_c1.log gpurun_out/ncu_c4.log; cat gpurun_out/skew24.jsonl gpurun_out/skew28.jsonl; tail -3 gpurun_out/skew28.err
