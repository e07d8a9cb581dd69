#!/bin/bash
# round 2au: k = 21..32 K-concatenated path with the GT fold: parity + configs
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_parity_gpu.py tests/test_configs_gpu.py tests/test_scale_gpu.py tests/test_solver_gpu.py -x -q > gpurun_out/r2au_pytest.log 2>&1
timeout 600 python tools/configs_probe.py > gpurun_out/r2au_configs.txt 2>&1
echo done
