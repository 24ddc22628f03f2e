#!/bin/bash
# alternating decode-step timings of several prebuilt libraries (ab/<name>.so): $1 = B, $2 = ctx, $3 = rounds, rest = names
B=$1; CTX=$2; R=$3; shift 3
for r in $(seq $R); do
  for v in "$@"; do
    echo -n "$v "; COCOB200_LIB=ab/$v.so timeout 300 python scripts/step_profile.py $B 5 $CTX 2>&1 | grep "decode step"
  done
done
