set -u
mkdir -p gpurun_out
for mp in 203 3203; do
timeout 300 ncu --set full --import-source on --clock-control none -k regex:gemm -s 3 -c 1 -o gpurun_out/qkv64_$mp -f python scripts/gemm_one.py 12288 4096 64 $mp > gpurun_out/ncu_q$mp.log 2>&1
done
