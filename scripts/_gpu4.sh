timeout 600 python -m pytest tests/test_kernels_gpu.py tests/test_model_gpu.py -q -x 2>&1 | tail -3 > gpurun_out/kt8.txt
for i in 1 2 3; do for B in 64 128; do timeout 300 python scripts/step_profile.py $B 20 2>&1 | head -1 | sed "s/^/kd2 /"; COCOB200_KD=1 timeout 300 python scripts/step_profile.py $B 20 2>&1 | head -1 | sed "s/^/kd1 /"; done; done > gpurun_out/step_kd2.txt
