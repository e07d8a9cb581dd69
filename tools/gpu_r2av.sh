#!/bin/bash
# round 2av: stacked G^T U for the KP16 = 64 split layout (A/B) + parity
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_scale_gpu.py -x -q > gpurun_out/r2av_pytest.log 2>&1
for r in 1 2; do for t in s0 s1; do
  echo "== $t round $r" >> gpurun_out/r2av_configs.txt
  SPCP_LIB_PATH=ab/lib_$t.so timeout 600 python tools/configs_probe.py >> gpurun_out/r2av_configs.txt 2>&1
done; done
echo done
