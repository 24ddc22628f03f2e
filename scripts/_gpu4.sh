timeout 120 python scripts/gemm_trace.py 12288 4096 256 0 6 0 > gpurun_out/trace11.txt 2>&1
timeout 120 python scripts/gemm_trace.py 22016 4096 256 0 6 3 >> gpurun_out/trace11.txt 2>&1
timeout 120 python scripts/gemm_trace.py 4096 4096 256 0 3 2 >> gpurun_out/trace11.txt 2>&1
