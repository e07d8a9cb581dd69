#!/bin/bash
# round 2z: stored-ray probes + fp32 probe cap: GPU tests, then the TTC trace
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_line_gpu.py tests/test_solver_gpu.py -x -q > gpurun_out/r2z_pytest.log 2>&1
timeout 900 python tools/ttc_trace_probe.py c2 c5 > gpurun_out/r2z_trace.log 2>&1
echo done
