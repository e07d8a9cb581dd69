#!/bin/bash
# round 2az: G^T U accumulator wait moved after the G.V issue (A/B) + parity
mkdir -p gpurun_out
tools/ab_run.sh gpurun_out/r2az_ab.txt 3 w0 w1
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_configs_gpu.py -x -q > gpurun_out/r2az_pytest.log 2>&1
echo done
