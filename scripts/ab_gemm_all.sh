#!/bin/bash
# A/B of ab/old.so vs ab/new.so: every decode projection at T = 1 .. 256 (real epilogues, fused norm), alternating
timeout 600 python -m pytest tests/test_kernels_gpu.py tests/test_headline_gpu.py -q -m gpu -x 2>&1 | tail -2
for r in 1 2; do
  for v in old new; do
    echo "== $v"
    COCOB200_LIB=ab/$v.so timeout 300 python scripts/gemm_perf.py 0 ${1:-256} --real-epi --norm 2>&1 | grep "T="
  done
done
