#!/bin/bash
# A/B of the decode attention positions in flight per lane group (u = 4 vs 8) for MHA with many CTAs, in-step
mkdir -p gpurun_out
run() { for B in 64 128 256; do python scripts/step_profile.py $B 10 256 2>/dev/null | head -1; done; }
echo "== u = 4 when >= 8 waves of CTAs (current)" > gpurun_out/ab_attn_u.txt; run >> gpurun_out/ab_attn_u.txt 2>&1
sed -i 's/const int u = gq == 1 \&\& total >= 8LL \* num_sms ? 4 : 8;/const int u = 8;/' paper_2507_18006_b200/csrc/attention.cu
python -c "from paper_2507_18006_b200 import _build; _build.build(force=True)" >> gpurun_out/ab_attn_u.txt 2>&1
echo "== u = 8 always" >> gpurun_out/ab_attn_u.txt; run >> gpurun_out/ab_attn_u.txt 2>&1
