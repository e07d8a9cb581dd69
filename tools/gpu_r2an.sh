#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_solver_gpu.py tests/test_dist_gpu.py -x -q > gpurun_out/r2an_pytest.log 2>&1
timeout 900 python tools/cert_c5_probe.py c5 > gpurun_out/r2an_cert.log 2>&1
echo done
