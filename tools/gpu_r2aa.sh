#!/bin/bash
# round 2aa: leader-polled S barrier in the epilogue (A/B), parity suite
mkdir -p gpurun_out
tools/ab_run.sh gpurun_out/r2aa_ab.txt 4 lw1 lw0
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_configs_gpu.py tests/test_scale_gpu.py -x -q > gpurun_out/r2aa_pytest.log 2>&1
echo done
