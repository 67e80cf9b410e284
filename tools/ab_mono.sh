#!/bin/bash
# monomial-route step (interpolate + full-width MSMs) under several settings
for e in "$@"; do echo "== $e $(env $e python tools/profile_mono.py 2>&1 | tail -1)"; done
