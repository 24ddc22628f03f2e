#!/bin/bash
timeout 600 python -m pytest tests/test_kernels_gpu.py tests/test_headline_gpu.py -q -m gpu -x 2>&1 | tail -2
bash scripts/ab_lib.sh
