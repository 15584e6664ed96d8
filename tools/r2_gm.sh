#!/bin/bash
# 32-bit modulo by invariant multiplier + unaligned-view histogram: timings and parity tests (GPU box)
mkdir -p gpurun_out
timeout 300 python tools/diag_hist.py 28 2>&1 | cut -c1-200
timeout 300 python tools/diag_vphase.py 2>&1 | cut -c1-250
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_fuzz_gpu.py tests/test_api_gpu.py tests/test_reference_suite_gpu.py tests/test_cli_gpu.py tests/test_skew_gpu.py tests/test_route_gpu.py tests/test_layout_gpu.py -q -m gpu -x -p no:cacheprovider 2>&1 | tail -2
