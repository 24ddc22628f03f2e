#!/bin/bash
# A/B of ab/old.so vs ab/new.so: O / down at T = 256 (real epilogues, fused norm) and the B = 256 step
timeout 600 python -m pytest tests/test_kernels_gpu.py tests/test_headline_gpu.py -q -m gpu -x 2>&1 | tail -2
for r in 1 2 3; do
  for v in old new; do
    echo "== $v"
    COCOB200_LIB=ab/$v.so timeout 300 python scripts/gemm_perf.py 0 256 --real-epi --norm 2>&1 | grep -E "^(o|down) "
  done
done
bash scripts/ab_step.sh 256 256 3
