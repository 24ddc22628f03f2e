for B in 64 256; do
timeout 300 python scripts/step_profile.py $B 3 > gpurun_out/step_$B.txt 2>&1
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch_$B.csv python scripts/step_profile.py $B 1 > /dev/null 2>&1
done
