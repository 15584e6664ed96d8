#!/bin/bash
# probe tail-unroll variants (GPU box): base = HG_TAIL_UNROLL 4
for v in "" tu1 tu2 tu8; do
  lib=""; [ -n "$v" ] && lib="HG_LIB=paper_2104_00792_b200/exp/$v.so"
  for a in "" "--load-factor 4" "--key-bits 64"; do
  env $lib timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 10 --warmup 3 $a 2>/dev/null | python tools/bench_line.py "[${v:-tu4} $a]" | cut -c1-110
  done
done
