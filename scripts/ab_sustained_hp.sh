#!/bin/bash
# sustained (power-capped) A/B: default vs SVD_HP=1, clocks sampled
for round in 1 2; do
 for hpv in 0 1; do
  nvidia-smi --query-gpu=clocks.sm,power.draw,clocks_event_reasons.sw_power_cap --format=csv,noheader -lms 200 > gpurun_out/clk_$hpv_$round.csv &
  CP=$!
  echo -n "SVD_HP=$hpv round $round: "
  SVD_HP=$hpv REPS=40 timeout 300 python scripts/time_layers.py hunyuan-dense hunyuan 2>&1 | tail -1
  kill $CP
  python3 -c "
import csv,statistics
r=[l for l in csv.reader(open('gpurun_out/clk_$hpv_$round.csv')) if l and 'MHz' in l[0]]
mhz=[float(x[0].split()[0]) for x in r]; w=[float(x[1].split()[0]) for x in r]
print('   clocks median', statistics.median(mhz), 'MHz, power median', statistics.median(w), 'W, samples', len(r))
"
 done
done
