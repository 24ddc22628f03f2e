#!/bin/bash
# A/B of the decode attention split target (MHA: 2 vs 4 waves of CTAs), in-step at small batches
mkdir -p gpurun_out
run() { for B in 4 16 32; do python scripts/step_profile.py $B 10 256 | head -1; done; }
echo "== want 2 waves (current)" > gpurun_out/ab_attn.txt; run >> gpurun_out/ab_attn.txt 2>&1
sed -i 's/const long long want = (gq > 1 ? 8LL : 2LL) \* num_sms;/const long long want = (gq > 1 ? 8LL : 4LL) * num_sms;/' paper_2507_18006_b200/csrc/attention.cu
python -c "from paper_2507_18006_b200 import _build; _build.build(force=True)" >> gpurun_out/ab_attn.txt 2>&1
echo "== want 4 waves" >> gpurun_out/ab_attn.txt; run >> gpurun_out/ab_attn.txt 2>&1
