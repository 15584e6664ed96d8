#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_layout_gpu.py tests/test_skew_gpu.py tests/test_gpu_parity.py tests/test_api_gpu.py -q -m gpu -x -p no:cacheprovider > gpurun_out/layout.log 2>&1; echo "rc=$?" >> gpurun_out/layout.log
tail -5 gpurun_out/layout.log
timeout 600 python tools/skew.py 30 uniform > gpurun_out/skew30.jsonl 2>gpurun_out/skew30.err; cat gpurun_out/skew30.jsonl; tail -2 gpurun_out/skew30.err
timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 10 --warmup 3 2>/dev/null | python tools/bench_line.py "[c1]" | cut -c1-200
