#!/bin/bash
# local-build capacity variants (GPU box): base = 38 keys per thread (19456 per bin)
for v in "" b44 b48; do
  lib=""; [ -n "$v" ] && lib="HG_LIB=paper_2104_00792_b200/exp/$v.so"
  for a in "" "--k 16"; do
  env $lib timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 10 --warmup 3 $a 2>/dev/null | python tools/bench_line.py "[${v:-b38} $a]" | cut -c1-190
  done
done
