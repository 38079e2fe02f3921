#!/bin/bash
# A/B kernel variants in one session, two interleaved rounds (clock drift).
V=paper_2506_03065_b200/variants
for round in 1 2; do
  for so in $V/*.so; do
    SVD_LIB=$PWD/$so timeout 120 python scripts/time_layers.py ${CONFIGS:-hunyuan cogvideo} 2>&1 | tail -1
  done
done
