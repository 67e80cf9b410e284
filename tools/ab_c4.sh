#!/bin/bash
# A/B of config-4 opening knobs (wall time of tc_open_many over the 256 challenges)
for e in "X=1" "TC_MSM_FP_MIN_N=65536" "TC_MSM_FP_MIN_N=16384" "TC_OPEN_PRECOMP_MIN=4" "TC_OPEN_PRECOMP_MIN=4 TC_MSM_FP_MIN_N=65536" "TC_OPEN_PRECOMP_MIN=3 TC_MSM_FP_MIN_N=65536"; do
  echo "== $e"
  env $e TC_C4_REPS=3 python tools/profile_c4.py 2>&1 | tail -2
done
