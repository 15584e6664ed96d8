#!/bin/bash
# query_sharded answers back through hg_reorganize_gather: parity tests + virtual-shard timings (GPU box)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_api_gpu.py tests/test_reference_suite_gpu.py tests/test_cli_gpu.py tests/test_multidevice_gpu.py tests/test_route_gpu.py -q -m gpu -x -p no:cacheprovider 2>&1 | tail -2
timeout 300 python tools/diag_vphase.py 2>&1 | cut -c1-300
