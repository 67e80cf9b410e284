#!/bin/bash
# rebuild the library (if any source changed), then run "$@" on the GPU box via gpurun
# usage: tools/gpu.sh TIMEOUT 'command'
set -e
cd /root/repo
python -c "from paper_2602_12630_b200 import build_ext; build_ext.build()" 2>&1 | tail -1
T=$1; shift
exec /usr/local/graft/bin/gpurun --timeout "$T" -- "$@"
