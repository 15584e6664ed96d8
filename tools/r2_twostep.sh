#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_two_step_gpu.py tests/test_gpu_parity.py tests/test_api_gpu.py -q -m gpu -x -p no:cacheprovider > gpurun_out/twostep.log 2>&1; echo "rc=$?" >> gpurun_out/twostep.log
tail -30 gpurun_out/twostep.log
timeout 600 python tools/two_step.py 28 2>&1 | tail -3
