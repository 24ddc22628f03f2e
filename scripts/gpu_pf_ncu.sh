#!/bin/bash
# ncu --set full of the current prefill attention kernel (one launch, 4 x 2048-token prompts)
mkdir -p gpurun_out
timeout 400 ncu --set full --clock-control none --import-source on -k regex:prefill_attn -c 1 -o gpurun_out/prof_pf_ptmem -f \
    python scripts/prefill_profile.py 4 2048 > gpurun_out/ncu_pf_ptmem.log 2>&1
ncu -i gpurun_out/prof_pf_ptmem.ncu-rep --page raw --csv > gpurun_out/pf_ptmem_raw.csv 2>/dev/null
