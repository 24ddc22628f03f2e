#!/bin/bash
# launch list of one decode step at batch 1 / 16 (ctx 256): where the small-batch step goes
mkdir -p gpurun_out
for B in 1 16; do
  timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/launches_b$B.csv python scripts/step_profile.py $B 1 256 > gpurun_out/ncu_b$B.log 2>&1
done
timeout 300 python scripts/step_profile.py 1 5 256 > gpurun_out/step_b1.txt 2>&1
