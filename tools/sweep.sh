#!/bin/bash
# tools/sweep.sh "ENV=.. ENV2=.." ... : times one MST per config under each env setting
for envs in "$@"; do
  for c in ${CONFIGS:-c1 c0 c2 c3}; do
    echo -n "[$envs] "; env $envs timeout 120 python tools/mst_once.py --config $c --warmup 2 --reps 5 2>&1 | grep "ms/MST\|rror" | tail -2
  done
done
