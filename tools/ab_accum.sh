#!/bin/bash
# A/B the bucket-accumulation kernel across library variants: bench.py per variant
for v in "$@"; do
  TC_LIB=$PWD/$v python bench.py --steps 5 --warmup 2 --no-cpu --no-forward --no-monomial 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['ms_per_step'],3), d['roofline']['work'].split('launches, ')[1], d['root'][:16])"
done
