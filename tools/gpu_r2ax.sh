#!/bin/bash
# round 2ax: G.V before G^T U in the reduction issuer (A/B) + parity
mkdir -p gpurun_out
tools/ab_run.sh gpurun_out/r2ax_ab.txt 3 o0 o1
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_configs_gpu.py -x -q > gpurun_out/r2ax_pytest.log 2>&1
echo done
