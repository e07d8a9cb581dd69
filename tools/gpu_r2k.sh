# round 2: sparse-observation passes with a round of gathers in flight
timeout 900 python -m pytest tests/test_sddmm_gpu.py -q > gpurun_out/r2k_sddmm.log 2>&1
timeout 1200 python tools/sddmm_probe.py > gpurun_out/r2k_sddmm_probe.log 2>&1
