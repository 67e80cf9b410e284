#!/bin/bash
# A/B of two library builds on the config-3 bench (alternating runs); build B with
# python -m paper_2602_12630_b200.build_ext --force --out=$PWD/_ab/lib_b.so -D...
for i in 1 2; do
  for lib in paper_2602_12630_b200/libtcb200.so _ab/lib_b.so; do
    echo "== $lib $(TC_LIB=$PWD/$lib python bench.py --steps 10 --warmup 3 --no-cpu --no-monomial 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d["ms_per_step"], d["e2e"]["value"])')"
  done
done
