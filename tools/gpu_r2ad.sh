#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_line_gpu.py -x -q > gpurun_out/r2ad_pytest.log 2>&1
timeout 600 python tools/line_bench.py > gpurun_out/r2ad_line.log 2>&1
echo done
