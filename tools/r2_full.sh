#!/bin/bash
# round-2 evidence pass: GPU suite, bench line, ncu launch list + full capture (GPU box)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider --durations=10 > gpurun_out/gputest.log 2>&1; echo "gpu tests rc=$?" >> gpurun_out/gputest.log
tail -15 gpurun_out/gputest.log
timeout 600 python bench.py --steps 10 --warmup 3 --cpu-log2 22 > gpurun_out/bench.log 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
python tools/bench_line.py "[bench]" < gpurun_out/bench.log | cut -c1-300
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name regex:"k_local_probe|k_local_build_p|k_part1|k_part2|k_unpart|k_hist" -c 12 -f -o gpurun_out/r2_full python tools/one_step.py 28 28 1.0 32 1 > gpurun_out/ncu_full.log 2>&1
tail -n 2 gpurun_out/ncu_full.log
