#!/bin/bash
# A/B environment settings on the config-3 bench: each argument is "VAR=val[,VAR=val]"
for spec in "$@"; do
  envs=$(echo "$spec" | tr ',' ' ')
  env $envs python bench.py --steps 5 --warmup 2 --no-cpu --no-forward --no-monomial 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$spec', round(d['ms_per_step'],3), d['roofline']['work'].split('launches, ')[1], d['root'][:16])"
done
