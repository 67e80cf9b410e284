#!/bin/bash
# sweep the window-plan parameters (TC_MSM_KAPPA:TC_MSM_CMAX pairs) on the config-3 bench
for kc in "$@"; do
  k=${kc%:*}; c=${kc#*:}
  TC_MSM_KAPPA=$k TC_MSM_CMAX=$c TC_MSM_DEBUG=1 python bench.py --steps 5 --warmup 2 --no-cpu --no-forward --no-monomial 2>/tmp/err.log | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('kappa:cmax $kc', round(d['ms_per_step'],3), d['roofline']['work'].split('launches, ')[1], d['root'][:16])"
  grep "L=32" /tmp/err.log | head -1
done
