#!/bin/bash
# A/B one env knob in one session, interleaved rounds (clock drift).
# usage: VAR=SVD_D64_KERNEL VALUES="tile half" CONFIGS="cogvideo" scripts/ab_env.sh
for round in 1 2; do
  for val in $VALUES; do
    echo -n "$VAR=$val "
    env $VAR=$val timeout 300 python scripts/time_layers.py ${CONFIGS:-cogvideo} 2>&1 | tail -1
  done
done
