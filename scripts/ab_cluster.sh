#!/bin/bash
# A/B: default two-tile kernel (cluster 4) vs one-tile double-buffered-S kernel (cluster 2)
V=paper_2506_03065_b200/variants
for round in 1 2; do
  SVD_CLUSTER=4 SVD_LIB=$PWD/$V/base.so timeout 120 python scripts/time_layers.py ${CONFIGS:-hunyuan cogvideo} | sed 's/^/c4 /'
  for so in base e1 e2 e3; do
    SVD_CLUSTER=2 SVD_LIB=$PWD/$V/$so.so timeout 120 python scripts/time_layers.py ${CONFIGS:-hunyuan cogvideo} | sed "s/^/c2 /"
  done
done
