#!/bin/bash
# round 2ar: G^T U drain with one TMEM wait per tile (A/B) + parity
mkdir -p gpurun_out
tools/ab_run.sh gpurun_out/r2ar_ab.txt 3 d0 d1
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_configs_gpu.py -x -q > gpurun_out/r2ar_pytest.log 2>&1
echo done
