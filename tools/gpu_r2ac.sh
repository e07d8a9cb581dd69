#!/bin/bash
# round 2ac: FP64 tensor-core k = 0 products (rSVD sketches): parity, init timing, TTC trace
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_solver_gpu.py tests/test_configs_gpu.py -x -q > gpurun_out/r2ac_pytest.log 2>&1
timeout 600 python tools/init_probe.py > gpurun_out/r2ac_init.log 2>&1
timeout 900 python tools/ttc_trace_probe.py c2 c5 > gpurun_out/r2ac_trace.log 2>&1
echo done
