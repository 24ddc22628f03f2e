#!/bin/bash
# A/B of two prebuilt libraries (ab/old.so, ab/new.so): O / down GEMMs at T = 256, the split-K timeline, the B = 256 step
for r in 1 2; do
  for v in old new; do
    echo "== $v"
    COCOB200_LIB=ab/$v.so timeout 300 python scripts/gemm_perf.py 0 256 --real-epi --norm 2>&1 | grep -E "^(o|down) "
    COCOB200_LIB=ab/$v.so timeout 300 python scripts/step_profile.py 256 3 256 2>&1 | grep "decode step"
  done
done
for v in old new; do echo "== trace $v"; COCOB200_LIB=ab/$v.so timeout 300 python scripts/gemm_split_trace.py 4096 4096 256 2>&1 | head -10; done
