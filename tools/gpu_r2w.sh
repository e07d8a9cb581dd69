#!/bin/bash
# round 2w: same-box A/B of the x-initialised residual accumulator, then the GPU suite
mkdir -p gpurun_out
tools/ab_run.sh gpurun_out/r2w_ab.txt 4 x1 x0
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2w_pytest.log 2>&1
echo done
