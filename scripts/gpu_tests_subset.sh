#!/bin/bash
# run a subset of the GPU tests with full output: $1 = pytest -k expression or test path list
mkdir -p gpurun_out
timeout 1200 python -m pytest $1 -q -x 2>&1 | tail -150 > gpurun_out/pytest_subset.txt
