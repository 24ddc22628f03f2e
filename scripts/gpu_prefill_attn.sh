set -u
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_kernels_gpu.py -k prefill -q -x 2>&1 | tail -5 > gpurun_out/pf_test.txt
timeout 900 python -m pytest tests/test_model_gpu.py tests/test_headline_gpu.py -q -x 2>&1 | tail -5 >> gpurun_out/pf_test.txt
for L in 128 512 2048; do B=$((8192 / L)); timeout 300 python scripts/prefill_profile.py $B $L >> gpurun_out/pf_perf.txt 2>&1; done
timeout 300 ncu --set full --clock-control none --import-source on -k regex:prefill_attn -c 1 -o gpurun_out/prof_pf -f python scripts/prefill_profile.py 4 2048 > gpurun_out/ncu_pf.log 2>&1
