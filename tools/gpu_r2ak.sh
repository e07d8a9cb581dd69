#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_solver_gpu.py tests/test_dist_gpu.py tests/test_scale_gpu.py tests/test_configs_gpu.py -q > gpurun_out/r2ak_pytest.log 2>&1
timeout 900 python tools/cert_c5_probe.py > gpurun_out/r2ak_cert.log 2>&1
timeout 900 python tools/cert_time_probe.py > gpurun_out/r2ak_cert_c2.log 2>&1
echo done
