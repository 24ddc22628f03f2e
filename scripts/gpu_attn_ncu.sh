#!/bin/bash
# ncu --set full of one TMA decode-attention launch (B = 256, ctx 256) + the step's launch list
mkdir -p gpurun_out
timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:attn_tma -c 1 \
  -o gpurun_out/prof_attn_tma -f python scripts/step_profile.py 256 1 256 > gpurun_out/ncu_attn_tma.log 2>&1
ncu -i gpurun_out/prof_attn_tma.ncu-rep --page raw --csv > gpurun_out/attn_tma_raw.csv 2>/dev/null
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_tma_256.csv python scripts/step_profile.py 256 1 256 > gpurun_out/ncu_launch_tma.log 2>&1
