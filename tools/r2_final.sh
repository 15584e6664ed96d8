#!/bin/bash
# final pass: smoke(), the whole -m gpu suite, one bench line (GPU box)
mkdir -p gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
tail -2 gpurun_out/smoke.log
timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider --durations=10 > gpurun_out/gputest.log 2>&1; echo "gpu tests rc=$?" >> gpurun_out/gputest.log
tail -6 gpurun_out/gputest.log
timeout 600 python bench.py > gpurun_out/bench_default.log 2> gpurun_out/bench_default.err; echo "bench rc=$?" >> gpurun_out/bench_default.err
python tools/bench_line.py "[bench]" < gpurun_out/bench_default.log | cut -c1-300
