#!/bin/bash
# A/B of config-4 opening knobs (wall time of tc_open_many over the 256 challenges)
for e in "$@"; do
  echo "== $e"
  env $e TC_C4_REPS=3 python tools/profile_c4.py 2>&1 | tail -2
done
