# round 2: fp64 register-blocked kernel: tests + timing
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r2d_pytest.log 2>&1
timeout 300 python tools/fp64_probe.py 10 > gpurun_out/r2d_fp64.log 2>&1
