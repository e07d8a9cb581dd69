# round 2: fp64 evaluation on DMMA: parity tests + timing
timeout 1200 python -m pytest tests/test_parity_gpu.py tests/test_scale_gpu.py tests/test_solver_gpu.py tests/test_sddmm_gpu.py -m gpu -q > gpurun_out/r2n_pytest.log 2>&1
timeout 300 python tools/fp64_probe.py 10 > gpurun_out/r2n_fp64.log 2>&1
