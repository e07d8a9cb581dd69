# round 2: final-state evidence: GPU suite, bench line, C5 shard probe, launch list, ncu of K1
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r2q_pytest.log 2>&1
timeout 1500 python bench.py > gpurun_out/r2q_bench.log 2>&1
timeout 900 python tools/c5_shard_probe.py > gpurun_out/r2q_c5_shards.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv \
  --log-file gpurun_out/r2q_launches.csv python bench.py --steps 5 --warmup 3 --skip-cpu --skip-e2e \
  --skip-ttc --skip-c5 > gpurun_out/r2q_ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_eval_kernel -s 30 -c 1 \
  -o gpurun_out/r2q_tc_full python bench.py --steps 5 --warmup 3 --skip-cpu --skip-e2e --skip-ttc \
  --skip-c5 > gpurun_out/r2q_ncu_full.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:tc_reduce -s 30 -c 1 \
  -o gpurun_out/r2q_reduce_full python bench.py --steps 5 --warmup 3 --skip-cpu --skip-e2e --skip-ttc \
  --skip-c5 > gpurun_out/r2q_ncu_reduce.log 2>&1
