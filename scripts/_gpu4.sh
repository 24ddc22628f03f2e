timeout 600 python -m pytest tests/test_model_gpu.py tests/test_kernels_gpu.py -q -x 2>&1 | tail -15 > gpurun_out/kt13.txt
for L in 128 512 2048; do timeout 300 python scripts/prefill_profile.py $((8192/L)) $L; done > gpurun_out/prefill2.txt 2>&1
