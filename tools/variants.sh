#!/bin/bash
# bench lines for the C=1 / C=4 / C3 / u64 variants, condensed (GPU box)
for args in "" "--load-factor 4" "--k 16" "--key-bits 64" ${EXTRA_VARIANTS}; do
  timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 10 --warmup 3 $args 2>/dev/null | python tools/bench_line.py "[${args:-c1}]"
done
