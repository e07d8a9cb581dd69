# round-2 probe: read-only HBM ceiling, and the fused kernel burst vs sustained
./tools/hbm_probe > gpurun_out/r2b_hbm.txt 2>&1
timeout 300 python bench.py --steps 20 --warmup 5 --skip-ttc --skip-cpu --skip-e2e > gpurun_out/r2b_b20.log 2>&1
timeout 300 python bench.py --steps 5000 --warmup 5 --skip-ttc --skip-cpu --skip-e2e > gpurun_out/r2b_b5000.log 2>&1
nvidia-smi -q -d CLOCK,POWER > gpurun_out/r2b_smi.txt 2>&1
