#!/bin/bash
# A/B of experimental library variants (GPU box): VARIANTS="name ..." (exp/<name>.so), "" = the built library
for v in "" ${VARIANTS}; do
  lib=""; [ -n "$v" ] && lib="HG_LIB=paper_2104_00792_b200/exp/$v.so"
  for a in "" "--load-factor 4" "--k 16" "--key-bits 64"; do
    env $lib timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 10 --warmup 3 $a 2>/dev/null | python tools/bench_line.py "[${v:-base} ${a}]" | cut -c1-200
  done
done
for v in ${VARIANTS}; do
  env HG_LIB=paper_2104_00792_b200/exp/$v.so timeout 900 python -m pytest -q -x -m gpu tests/test_fuzz_gpu.py tests/test_skew_gpu.py tests/test_gpu_parity.py 2>&1 | tail -2
done
