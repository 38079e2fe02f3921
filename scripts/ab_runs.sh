#!/bin/bash
# A/B arbitrary (env, library) runs in one session, interleaved rounds.
# usage: CONFIGS="cogvideo" scripts/ab_runs.sh "SVD_LIB=a.so" "SVD_LIB=b.so SVD_D64_KERNEL=tile" ...
for round in 1 2; do
  for run in "$@"; do
    echo -n "[$run] "
    env $run timeout 300 python scripts/time_layers.py ${CONFIGS:-cogvideo} 2>&1 | tail -1
  done
done
