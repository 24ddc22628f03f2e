#!/bin/bash
# One GPU session: parity tests, smoke, bench, ncu launch list + full captures.
set -u
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.used --format=csv > $OUT/gpu.txt 2>&1
if [ "${SKIP_TESTS:-0}" != "1" ]; then
  timeout 900 python -m pytest tests -m gpu -q -rA 2>&1 | tail -60 > $OUT/pytest_gpu.txt
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.txt 2>&1
fi
timeout 900 python bench.py ${BENCH_ARGS:-} > $OUT/bench.json 2> $OUT/bench.err
if [ "${SKIP_NCU:-0}" != "1" ]; then
  for B in 64 256; do
    # every launch of one decode step (cudaProfilerStart/Stop brackets it): cold-cache, serialised
    timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
        --log-file $OUT/launches_$B.csv python scripts/step_profile.py $B 1 ${CTX:-256} > $OUT/ncu_launch_$B.log 2>&1
    # full sections of the four decode GEMMs of layer 1 and its attention
    timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:gemm -c 4 \
        -o $OUT/prof_gemm_$B -f python scripts/step_profile.py $B 1 ${CTX:-256} > $OUT/ncu_gemm_$B.log 2>&1
    timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:attn2 -c 1 \
        -o $OUT/prof_attn_$B -f python scripts/step_profile.py $B 1 ${CTX:-256} > $OUT/ncu_attn_$B.log 2>&1
  done
fi
ls -la $OUT
