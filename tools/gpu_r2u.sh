# round 2: final bench line + reference arm (driver-like arguments) + configs probe
timeout 1500 python bench.py > gpurun_out/r2u_bench.log 2>&1
timeout 900 python tools/configs_probe.py > gpurun_out/r2u_configs.log 2>&1
timeout 1500 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r2u_ref.log 2>&1
