#!/bin/bash
# skew parity + GPU suite + skew timings + a short bench line (GPU box)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_skew_gpu.py -q -m gpu -x -p no:cacheprovider --durations=8 > gpurun_out/skewtest.log 2>&1; echo "skew tests rc=$?" >> gpurun_out/skewtest.log
tail -15 gpurun_out/skewtest.log
if [ -z "$QUICK" ]; then
timeout 900 python -m pytest tests -q -m gpu -x -p no:cacheprovider --ignore=tests/test_scale_parity_gpu.py --ignore=tests/test_skew_gpu.py > gpurun_out/gputest.log 2>&1; echo "gpu tests rc=$?" >> gpurun_out/gputest.log
tail -5 gpurun_out/gputest.log
fi
timeout 600 python tools/skew.py 28 > gpurun_out/skew28.jsonl 2> gpurun_out/skew28.err; echo "skew28 rc=$?" >> gpurun_out/skew28.err
cat gpurun_out/skew28.jsonl; tail -3 gpurun_out/skew28.err
bash tools/variants.sh 2>&1 | tee gpurun_out/variants.txt
