#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_kernels_gpu.py tests/test_model_gpu.py tests/test_headline_gpu.py -q -x 2>&1 | tail -5 > gpurun_out/attn_test.txt
for B in 1 4 16; do timeout 300 python scripts/step_profile.py $B 5 256; done > gpurun_out/attn_steps.txt 2>&1
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_b1.csv python scripts/step_profile.py 1 1 256 > gpurun_out/ncu_b1.log 2>&1
