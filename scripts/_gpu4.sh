timeout 600 python -m pytest tests/test_kernels_gpu.py tests/test_model_gpu.py -q -x 2>&1 | tail -15 > gpurun_out/kt11.txt
timeout 300 python scripts/gemm_perf.py 0 8,64,128 --real-epi > gpurun_out/perf_cs.txt 2>&1
COCOB200_CSTREAM=0 timeout 300 python scripts/gemm_perf.py 0 8,64,128 --real-epi > gpurun_out/perf_nocs.txt 2>&1
for i in 1 2; do for B in 64 128; do timeout 300 python scripts/step_profile.py $B 20 2>&1 | head -1 | sed "s/^/cs   /"; COCOB200_CSTREAM=0 timeout 300 python scripts/step_profile.py $B 20 2>&1 | head -1 | sed "s/^/nocs /"; done; done > gpurun_out/step_cs.txt
