#!/bin/bash
# pipelined step / e2e / lone-forward latency for several library builds (TC_LIB), alternating:
#   ab_libs_lat.sh lib1.so lib2.so ...
for i in 1 2; do
  for lib in "$@"; do
    echo "== $lib $(TC_LIB=$PWD/$lib python bench.py --steps 40 --warmup 5 --no-cpu --no-forward --no-monomial 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["ms_per_step"],4), round(d["e2e"]["ms_per_step"],4), round(d["latency_ms"],4))')"
  done
done
