#!/bin/bash
# On the GPU box: GPU tests + u32/u64/high-dup bench lines with the per-kernel breakdown.
# usage (here): tools/gpu.sh 900 'bash tools/gpu_check.sh'
timeout 700 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
for args in "--key-bits 32" "--key-bits 64" "--k 16"; do
  timeout 300 python bench.py $args --no-cpu-baseline --no-e2e --steps 10 --warmup 3 2>&1 | grep "^{" | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$args', round(d['value']/1e9,3), 'G keys/s', round(d['ms_per_step'],3), 'ms')
print('  ' + ', '.join(f\"{k['kernel']} {k['avg_ms']:.3f}\" for k in d['kernels'][:10]))"
done
