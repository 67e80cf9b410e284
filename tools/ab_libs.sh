#!/bin/bash
# config-3 bench (pipelined step and e2e) for several library builds (TC_LIB), alternating:
#   ab_libs.sh lib1.so lib2.so ...
for i in 1 2; do
  for lib in "$@"; do
    echo "== $lib $(TC_LIB=$PWD/$lib python bench.py --steps 10 --warmup 3 --no-cpu --no-monomial 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["ms_per_step"],3), round(d["e2e"]["ms_per_step"],3), d["roofline"]["work"][-10:])')"
  done
done
