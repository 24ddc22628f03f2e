#!/bin/bash
# A/B of two prebuilt libraries (ab/old.so, ab/new.so) on the 7B decode step: alternating runs
B=${1:-256}; CTX=${2:-256}; R=${3:-4}
for r in $(seq $R); do
  for v in old new; do
    echo -n "$v "; COCOB200_LIB=ab/$v.so timeout 300 python scripts/step_profile.py $B 5 $CTX 2>&1 | grep "decode step"
  done
done
