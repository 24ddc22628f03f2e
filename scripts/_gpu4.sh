timeout 600 python -m pytest tests/test_kernels_gpu.py -q -x 2>&1 | tail -3 > gpurun_out/kt4.txt
timeout 300 python scripts/gemm_perf.py 0 64,256 --real-epi > gpurun_out/perf_epi3.txt 2>&1
for B in 64 256; do timeout 300 python scripts/step_profile.py $B 3 > gpurun_out/step_$B.txt 2>&1; done
