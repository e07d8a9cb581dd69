# round 2: tests (all), A/B of the fused prep kernel, ncu launch list + full capture of K1
timeout 1800 python -m pytest tests -m gpu -q -s > gpurun_out/r2g_pytest.log 2>&1
tools/ab_run.sh gpurun_out/r2g_ab.log 2 prep0 prep1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv \
  --log-file gpurun_out/r2g_launches.csv python bench.py --steps 5 --warmup 3 --skip-cpu --skip-e2e \
  --skip-ttc --skip-c5 > gpurun_out/r2g_ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_eval_kernel -s 30 -c 1 \
  -o gpurun_out/r2g_tc_full python bench.py --steps 5 --warmup 3 --skip-cpu --skip-e2e --skip-ttc \
  --skip-c5 > gpurun_out/r2g_ncu_full.log 2>&1
