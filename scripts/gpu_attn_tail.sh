#!/bin/bash
timeout 900 python -m pytest tests/test_kernels_gpu.py tests/test_headline_gpu.py -q -m gpu -x 2>&1 | tail -2
bash scripts/ab_step_multi.sh 256 270 3 old new
bash scripts/ab_step_multi.sh 256 256 2 old new
