for i in 1 2; do
for B in 64 256; do timeout 300 python scripts/step_profile.py $B 5 2>&1 | head -1; COCOB200_NO_TMA_STORE=1 timeout 300 python scripts/step_profile.py $B 5 2>&1 | head -1; done
done > gpurun_out/ab_tma.txt
