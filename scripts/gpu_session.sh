#!/bin/bash
# Ad-hoc GPU session: the tests and measurements named in $1 (comma list).
set -u
mkdir -p gpurun_out
IFS=',' read -ra JOBS <<< "${1:-}"
for j in "${JOBS[@]}"; do
  case $j in
    pftest) timeout 600 python -m pytest tests/test_kernels_gpu.py -k prefill -q -x 2>&1 | tail -5 > gpurun_out/pf_test.txt
            timeout 600 python -m pytest tests/test_model_gpu.py -k "prefill" -q -x 2>&1 | tail -5 >> gpurun_out/pf_test.txt ;;
    pfperf) for L in 128 512 2048 4096; do B=$((8192 / L)); timeout 300 python scripts/prefill_profile.py $B $L; done > gpurun_out/pf_perf.txt 2>&1 ;;
    pfncu) timeout 300 ncu --set full --clock-control none --import-source on -k regex:prefill_attn -c 1 \
             -o gpurun_out/prof_pf -f python scripts/prefill_profile.py 4 2048 > gpurun_out/ncu_pf.log 2>&1 ;;
    gemmod) timeout 600 python scripts/gemm_perf.py 0,352,354 16,64,96,128 --real-epi --norm > gpurun_out/gemm_od.txt 2>&1 ;;
    gputests) timeout 1800 python -m pytest tests -m gpu -q -rA 2>&1 | tail -60 > gpurun_out/pytest_gpu.txt ;;
    smoke) timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print(\"smoke ok\")" > gpurun_out/smoke.txt 2>&1 ;;
    bench) timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err ;;
    configs) timeout 900 python scripts/config3_replication.py --out gpurun_out/config3.json > gpurun_out/config3.log 2>&1
             timeout 900 python scripts/config4_migration.py --out gpurun_out/config4.json > gpurun_out/config4.log 2>&1
             timeout 900 python scripts/config5_70b_sharded.py --out gpurun_out/config5.json > gpurun_out/config5.log 2>&1 ;;
    gemmsmall) timeout 600 python scripts/gemm_perf.py 0,2,3,4,99 1,16 --real-epi --norm > gpurun_out/gemm_small.txt 2>&1 ;;
  esac
done
ls gpurun_out
