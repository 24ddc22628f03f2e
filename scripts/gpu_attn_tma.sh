#!/bin/bash
timeout 900 python -m pytest tests/test_headline_gpu.py tests/test_model_gpu.py -q -m gpu -x 2>&1 | tail -3
bash scripts/ab_step.sh 256 256 3
bash scripts/ab_step.sh 64 256 2
