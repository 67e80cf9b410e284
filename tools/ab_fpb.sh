#!/bin/bash
# A/B of the mode-1 counting sort: block-private counters (scatter LG MSMs per launch) vs global atomics
for e in "TC_MSM_FPB_LG=8" "TC_MSM_FPB_LG=4" "TC_MSM_FPB_LG=12" "TC_MSM_FPB_LG=16" "TC_MSM_NO_BLKCNT=1" "TC_MSM_FPB_LG=8"; do
  echo "== $e $(env $e python bench.py --steps 10 --warmup 3 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d["ms_per_step"], d["e2e"]["value"])')"
done
