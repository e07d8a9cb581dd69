#!/bin/bash
# round 2aj: certificate gradient route + stored G: tests + C5 certificate timing
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_solver_gpu.py tests/test_dist_gpu.py tests/test_scale_gpu.py -x -q > gpurun_out/r2aj_pytest.log 2>&1
timeout 900 python tools/cert_c5_probe.py > gpurun_out/r2aj_cert.log 2>&1
echo done
