#!/bin/bash
# round 2ba: final-state evidence (final fused kernel): GPU suite, bench line, configs, C5 shards,
# launch list, ncu --set full of the fused kernel and the reduce (exported to
# CSV on the box; only the fused kernel's report is kept: gpurun_out <= 64 MiB),
# reference arm
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r2ba_pytest.log 2>&1
timeout 1500 python bench.py > gpurun_out/r2ba_bench.log 2>&1
timeout 900 python tools/configs_probe.py > gpurun_out/r2ba_configs.log 2>&1
timeout 900 python tools/c5_shard_probe.py > gpurun_out/r2ba_c5_shards.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv \
  --log-file gpurun_out/r2ba_launches.csv python bench.py --steps 5 --warmup 3 --skip-cpu --skip-e2e \
  --skip-ttc --skip-c5 > gpurun_out/r2ba_ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_eval_kernel -s 30 -c 1 \
  -o gpurun_out/r2ba_tc_full python bench.py --steps 5 --warmup 3 --skip-cpu --skip-e2e --skip-ttc \
  --skip-c5 > gpurun_out/r2ba_ncu_full.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:tc_reduce -s 30 -c 1 \
  -o /tmp/r2ba_reduce_full python bench.py --steps 5 --warmup 3 --skip-cpu --skip-e2e --skip-ttc \
  --skip-c5 > gpurun_out/r2ba_ncu_reduce.log 2>&1
ncu -i /tmp/r2ba_reduce_full.ncu-rep --page raw --csv > gpurun_out/r2ba_reduce_raw.csv 2>&1
ncu -i gpurun_out/r2ba_tc_full.ncu-rep --page raw --csv > gpurun_out/r2ba_tc_raw.csv 2>&1
timeout 1500 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r2ba_ref.log 2>&1
du -sh gpurun_out
echo done
