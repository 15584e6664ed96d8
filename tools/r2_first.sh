#!/bin/bash
# round-2 first GPU pass: full GPU suite, scale parity, one bench line
mkdir -p gpurun_out
nproc > gpurun_out/host.txt; free -g >> gpurun_out/host.txt; lscpu | grep "Model name" >> gpurun_out/host.txt
timeout 900 python -m pytest tests -q -m gpu --ignore=tests/test_scale_parity_gpu.py -p no:cacheprovider > gpurun_out/gputest.log 2>&1; echo "gpu tests rc=$?" >> gpurun_out/gputest.log
timeout 1200 python -m pytest tests/test_scale_parity_gpu.py -q -m gpu -p no:cacheprovider --durations=0 > gpurun_out/scale.log 2>&1; echo "scale rc=$?" >> gpurun_out/scale.log
timeout 600 python bench.py --steps 10 --warmup 3 --cpu-log2 22 > gpurun_out/bench.log 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
tail -3 gpurun_out/gputest.log; tail -3 gpurun_out/scale.log; tail -2 gpurun_out/bench.err
