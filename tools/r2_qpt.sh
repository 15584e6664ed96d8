#!/bin/bash
# probe batch-size variants (GPU box): base = QPT 4 (u32) / 8 (u64)
for v in "" q6 q8; do
  lib=""; [ -n "$v" ] && lib="HG_LIB=paper_2104_00792_b200/exp/$v.so"
  for a in "" "--load-factor 4"; do
  env $lib timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 10 --warmup 3 $a 2>/dev/null | python tools/bench_line.py "[${v:-base} $a]" | cut -c1-110
  done
done
for v in "" q64_6 q64_12; do
  lib=""; [ -n "$v" ] && lib="HG_LIB=paper_2104_00792_b200/exp/$v.so"
  env $lib timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 10 --warmup 3 --key-bits 64 2>/dev/null | python tools/bench_line.py "[${v:-base} u64]" | cut -c1-110
done
