#!/bin/bash
# round 2bb: G.V on an early TMEM barrier (A/B) + parity
mkdir -p gpurun_out
tools/ab_run.sh gpurun_out/r2bb_ab.txt 3 e0 e1
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_configs_gpu.py -x -q > gpurun_out/r2bb_pytest.log 2>&1
echo done
