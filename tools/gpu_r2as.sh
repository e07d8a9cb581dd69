#!/bin/bash
# round 2as: K-concatenated layout for k = 21..32 (one-atom rows, re-read third
# segment): parity, then configs probe KC vs split (SPCP_TC_LAYOUT=split)
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_parity_gpu.py tests/test_configs_gpu.py tests/test_scale_gpu.py tests/test_sddmm_gpu.py -x -q > gpurun_out/r2as_pytest.log 2>&1
for r in 1 2; do
  echo "== kc round $r" >> gpurun_out/r2as_configs.txt
  timeout 600 python tools/configs_probe.py >> gpurun_out/r2as_configs.txt 2>&1
  echo "== split round $r" >> gpurun_out/r2as_configs.txt
  SPCP_TC_LAYOUT=split timeout 600 python tools/configs_probe.py >> gpurun_out/r2as_configs.txt 2>&1
done
echo done
