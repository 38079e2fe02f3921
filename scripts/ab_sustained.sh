#!/bin/bash
# sustained (power-capped) A/B of env settings, clocks / power sampled
# usage: scripts/ab_sustained.sh "ENV1" "ENV2" ...   (REPS, CONFIGS env)
for round in 1 2; do
 for run in "$@"; do
  nvidia-smi --query-gpu=clocks.sm,power.draw --format=csv,noheader -lms 200 > gpurun_out/clk_tmp.csv &
  CP=$!
  echo -n "[$run] round $round: "
  env $run REPS=${REPS:-40} timeout 400 python scripts/time_layers.py ${CONFIGS:-hunyuan-dense hunyuan} 2>&1 | tail -1
  kill $CP
  python3 -c "
import csv,statistics
r=[l for l in csv.reader(open('gpurun_out/clk_tmp.csv')) if l and 'MHz' in l[0]]
mhz=[float(x[0].split()[0]) for x in r]; w=[float(x[1].split()[0]) for x in r]
print('   clocks median', statistics.median(mhz), 'MHz, power median', statistics.median(w), 'W, samples', len(r))
"
 done
done
