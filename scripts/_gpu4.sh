timeout 600 python -m pytest tests/test_kernels_gpu.py tests/test_model_gpu.py -q -x 2>&1 | tail -3 > gpurun_out/kt9.txt
for i in 1 2; do for B in 64 128; do timeout 300 python scripts/step_profile.py $B 20 2>&1 | head -1 | sed "s/^/corun /"; COCOB200_CORUN=0 timeout 300 python scripts/step_profile.py $B 20 2>&1 | head -1 | sed "s/^/base  /"; done; done > gpurun_out/step_corun.txt
timeout 300 python scripts/gemm_perf.py 0 64,128 --real-epi > gpurun_out/perf_corun.txt 2>&1
