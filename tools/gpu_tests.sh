#!/bin/bash
# GPU pass: named test files (default: the whole -m gpu suite minus the scale tests), logs under gpurun_out/
mkdir -p gpurun_out
files=${@:-tests}
timeout 2400 python -m pytest $files -q -m gpu -p no:cacheprovider --ignore=tests/test_scale_parity_gpu.py --durations=15 -x > gpurun_out/gputest.log 2>&1
echo "gpu tests rc=$?" >> gpurun_out/gputest.log
tail -25 gpurun_out/gputest.log
