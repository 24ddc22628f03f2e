#!/bin/bash
# Interleaved A/B of one decode step (scripts/step_profile.py), R rounds:
#   bash scripts/ab_step.sh B R "ENV_A" "ENV_B"   (ENV_* = "" or "VAR=1 VAR2=1")
B=$1; R=${2:-3}; A=$3; BB=$4
for r in $(seq $R); do
  echo "A $(env $A timeout 300 python scripts/step_profile.py $B 10 2>&1 | head -1)"
  echo "B $(env $BB timeout 300 python scripts/step_profile.py $B 10 2>&1 | head -1)"
done
