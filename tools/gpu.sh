#!/bin/bash
# Rebuild the library in-tree, then run a command on the GPU box.
# usage: tools/gpu.sh TIMEOUT 'command'
set -e
cd /root/repo
python -m paper_2104_00792_b200._build --force > /tmp/build.log 2>&1 || { tail -30 /tmp/build.log; exit 1; }
/usr/local/graft/bin/gpurun --timeout "$1" -- "$2"
