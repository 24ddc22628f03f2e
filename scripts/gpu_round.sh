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
  # every launch of two timed decode steps (cold-cache, serialised: compare shares)
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 588 -c 260 --csv \
      --log-file $OUT/launches.csv python bench.py --batch 64 --sweep '' --steps 2 --warmup 1 --no-cpu-baseline --serve-s 0 > $OUT/ncu_launch.log 2>&1
  # full sections of the decode GEMMs (qkv, o, gate/up, down) and attention
  # decode GEMMs of the timed step (skip the lm_head of prefill + the warm-up step's 129)
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_tc_kernel -s 130 -c 4 \
      -o $OUT/prof_gemm -f python bench.py --batch 64 --sweep '' --steps 1 --warmup 1 --no-cpu-baseline --serve-s 0 > $OUT/ncu_gemm.log 2>&1
  # prefill GEMMs of layer 1 (T = 64 x 128 = 8192 rows): the tensor-bound case
  timeout 900 ncu --set full --clock-control none -k regex:gemm_tc2 -s 0 -c 4 \
      -o $OUT/prof_prefill -f python bench.py --batch 64 --sweep '' --steps 1 --warmup 1 --no-cpu-baseline --serve-s 0 > $OUT/ncu_prefill.log 2>&1
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_kernel -s 64 -c 1 \
      -o $OUT/prof_attn -f python bench.py --batch 64 --sweep '' --steps 1 --warmup 1 --no-cpu-baseline --serve-s 0 > $OUT/ncu_attn.log 2>&1
fi
ls -la $OUT
