#!/bin/bash
# round 2be: the N > 1 code path end to end with both ranks on one GPU (gloo):
# sharded evaluation, sharded C5 solve (stored-ray probes per shard) and certificate
mkdir -p gpurun_out
timeout 1500 python bench.py --gpus 2 --backend gloo --steps 10 --warmup 3 --skip-cpu --skip-e2e > gpurun_out/r2be_bench2.log 2>&1
echo "rc=$?" >> gpurun_out/r2be_bench2.log
echo done
