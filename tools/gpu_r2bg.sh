#!/bin/bash
# round 2bg: fold kernel on by default above 2^24 entries: GPU suite, smoke, bench
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r2bg_pytest.log 2>&1
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r2bg_smoke.log 2>&1
timeout 1500 python bench.py > gpurun_out/r2bg_bench.log 2>&1
timeout 600 python tools/configs_probe.py > gpurun_out/r2bg_configs.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv \
  --log-file gpurun_out/r2bg_launches.csv python bench.py --steps 5 --warmup 3 --skip-cpu --skip-e2e \
  --skip-ttc --skip-c5 > gpurun_out/r2bg_ncu_launch.log 2>&1
echo done
