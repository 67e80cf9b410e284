#!/bin/bash
# config-3 bench under a list of environment settings (knob sweeps): ab_env.sh "A=1" "B=2 C=3" ...
for e in "$@"; do
  echo "== $e $(env $e python bench.py --steps 10 --warmup 3 --no-cpu --no-monomial 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d["ms_per_step"], d["e2e"]["value"])')"
done
