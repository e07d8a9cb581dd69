#!/bin/bash
mkdir -p gpurun_out
timeout 600 python tools/line_bench.py > gpurun_out/r2z2_line.log 2>&1
timeout 600 python -m pytest tests/test_line_gpu.py tests/test_dist_gpu.py -x -q > gpurun_out/r2z2_pytest.log 2>&1
timeout 900 python tools/ttc_trace_probe.py c2 c5 > gpurun_out/r2z2_trace.log 2>&1
echo done
