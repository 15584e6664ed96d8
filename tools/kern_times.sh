#!/bin/bash
# usage (GPU box): bash tools/kern_times.sh LABEL [bench args...] -- prints the per-kernel avg ms
label=$1; shift
timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 5 --warmup 3 "$@" 2>&1 | grep "^{" | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$label', round(d['value']/1e9,3), 'G/s', round(d['ms_per_step'],3), 'ms |', ', '.join(f\"{k['kernel']} {k['avg_ms']:.3f}\" for k in d['kernels'][:9]))"
