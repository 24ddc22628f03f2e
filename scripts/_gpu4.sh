timeout 600 python -m pytest tests/test_kernels_gpu.py tests/test_model_gpu.py -q -x 2>&1 | tail -15 > gpurun_out/kt10.txt
timeout 300 python scripts/attn_perf.py > gpurun_out/attn_v2.txt 2>&1
CB_ATTN_V1=1 timeout 300 python scripts/attn_perf.py > gpurun_out/attn_v1.txt 2>&1
for B in 64 256; do timeout 300 python scripts/step_profile.py $B 20 2>&1 | head -1 | sed "s/^/v2 /"; CB_ATTN_V1=1 timeout 300 python scripts/step_profile.py $B 20 2>&1 | head -1 | sed "s/^/v1 /"; done > gpurun_out/step_attn.txt
