#!/bin/bash
# round 2at: GT fold (64-row G^T U slots) with the k = 21..32 K-concatenated path
mkdir -p gpurun_out
for r in 1 2; do for t in f0 f1; do
  echo "== $t round $r" >> gpurun_out/r2at_configs.txt
  SPCP_LIB_PATH=ab/lib_$t.so timeout 600 python tools/configs_probe.py >> gpurun_out/r2at_configs.txt 2>&1
done; done
echo "== split" >> gpurun_out/r2at_configs.txt
SPCP_TC_LAYOUT=split SPCP_LIB_PATH=ab/lib_f0.so timeout 600 python tools/configs_probe.py >> gpurun_out/r2at_configs.txt 2>&1
timeout 900 python -m pytest tests/test_parity_gpu.py -x -q > gpurun_out/r2at_pytest.log 2>&1
echo done
