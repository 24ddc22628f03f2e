#!/bin/bash
# A/B: attention pulling the O projection's weights into L2 at small batches (current build) vs without
mkdir -p gpurun_out
run() { for B in 1 4 16 32 64; do python scripts/step_profile.py $B 10 256 2>/dev/null | head -1; done; }
echo "== with the L2 prefetch of Wo during attention (T <= 32)" > gpurun_out/ab_l2.txt; run >> gpurun_out/ab_l2.txt 2>&1
sed -i 's/constexpr int kL2PrefetchRows = 32;/constexpr int kL2PrefetchRows = 0;/' paper_2507_18006_b200/csrc/runtime.cu
python -c "from paper_2507_18006_b200 import _build; _build.build(force=True)" >> gpurun_out/ab_l2.txt 2>&1
echo "== without" >> gpurun_out/ab_l2.txt; run >> gpurun_out/ab_l2.txt 2>&1
