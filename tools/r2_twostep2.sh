#!/bin/bash
# two-step: default library vs the HG_TRACE_DIRECT variant -- tests + device times (GPU box)
mkdir -p gpurun_out
for lib in "" paper_2104_00792_b200/exp/tdirect.so; do
  echo "== lib ${lib:-default}"
  HG_LIB=$lib timeout 900 python -m pytest tests/test_two_step_gpu.py tests/test_api_gpu.py -q -m gpu -x -p no:cacheprovider 2>&1 | tail -2
  HG_LIB=$lib timeout 600 python tools/two_step.py 28 2>&1 | tail -2
done 2>&1 | tee gpurun_out/twostep2.log
