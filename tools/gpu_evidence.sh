#!/bin/bash
# One GPU-box pass that produces the round's evidence:
#   pytest -m gpu, a full bench line, the ncu launch list of the same bench
#   command, and one `ncu --set full` capture of the fused streaming kernel.
# Usage (from the repo root, on the box): bash tools/gpu_evidence.sh TAG
TAG=${1:-r01}
O=gpurun_out
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/${TAG}_smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $O/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc $?" >> $O/${TAG}_pytest_gpu.log
timeout 600 python bench.py > $O/${TAG}_bench.log 2>&1; echo "bench rc $?" >> $O/${TAG}_bench.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $O/${TAG}_launches.csv python bench.py --steps 3 --warmup 3 --skip-cpu --skip-e2e --skip-ttc \
  > $O/${TAG}_ncu_launch.log 2>&1; echo "ncu launch rc $?" >> $O/${TAG}_ncu_launch.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_eval_kernel -s 4 -c 1 \
  -o $O/${TAG}_tc_full python bench.py --steps 3 --warmup 3 --skip-cpu --skip-e2e --skip-ttc \
  > $O/${TAG}_ncu_full.log 2>&1; echo "ncu full rc $?" >> $O/${TAG}_ncu_full.log
