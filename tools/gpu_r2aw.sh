#!/bin/bash
# round 2aw: final state after the k = 21..32 path and the Gram pass: GPU suite,
# bench line, configs, C5 shards, reference arm
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r2aw_pytest.log 2>&1
timeout 1500 python bench.py > gpurun_out/r2aw_bench.log 2>&1
timeout 900 python tools/configs_probe.py > gpurun_out/r2aw_configs.log 2>&1
timeout 900 python tools/c5_shard_probe.py > gpurun_out/r2aw_c5_shards.log 2>&1
timeout 1500 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r2aw_ref.log 2>&1
echo done
