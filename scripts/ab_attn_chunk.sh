#!/bin/bash
# A/B of the decode attention's minimum context chunk per split (MHA) at small batches, in-step
mkdir -p gpurun_out
run() { for B in 1 2 4 8; do python scripts/step_profile.py $B 10 256 2>/dev/null | head -1; done; }
: > gpurun_out/ab_chunk.txt
for C in 64 128 256 32; do
  sed -i "s/const int min_chunk = gq > 1 ? 128 : [0-9]*;/const int min_chunk = gq > 1 ? 128 : $C;/" paper_2507_18006_b200/csrc/attention.cu
  python -c "from paper_2507_18006_b200 import _build; _build.build(force=True)" >> gpurun_out/ab_chunk.txt 2>&1
  echo "== min_chunk $C" >> gpurun_out/ab_chunk.txt; run >> gpurun_out/ab_chunk.txt 2>&1
done
