#!/bin/bash
# round 2bf: one-block-per-segment fold kernel (SPCP_TC_FOLD=1) vs the LPI fold, all configs
mkdir -p gpurun_out
for r in 1 2; do
  echo "== lpi round $r" >> gpurun_out/r2bf_configs.txt
  timeout 600 python tools/configs_probe.py >> gpurun_out/r2bf_configs.txt 2>&1
  echo "== fold round $r" >> gpurun_out/r2bf_configs.txt
  SPCP_TC_FOLD=1 timeout 600 python tools/configs_probe.py >> gpurun_out/r2bf_configs.txt 2>&1
done
echo done
