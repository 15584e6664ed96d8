#!/bin/bash
# level-2 partition / local build grouped over level-1 bins (L2 residency experiment)
for g in 0 2 4 8 16; do
  HG_GROUPED=$g timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 10 --warmup 3 2>/dev/null | python tools/bench_line.py "[grouped $g]" | cut -c1-200
done
HG_GROUPED=4 timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_skew_gpu.py -q -m gpu -x -p no:cacheprovider 2>&1 | tail -1
