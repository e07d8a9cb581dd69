#!/bin/bash
mkdir -p gpurun_out
timeout 600 python tools/line_bench.py > gpurun_out/r2ab_line.log 2>&1
timeout 600 python -m pytest tests/test_line_gpu.py -x -q > gpurun_out/r2ab_pytest.log 2>&1
timeout 900 python tools/cert_c5_probe.py > gpurun_out/r2ab_cert.log 2>&1
echo done
