# round 2: floating G split (precision at small residuals): config tests + dist test, A/B timing
timeout 1800 python -m pytest tests/test_configs_gpu.py tests/test_dist_gpu.py tests/test_parity_gpu.py tests/test_scale_gpu.py -m gpu -q -s > gpurun_out/r2h_pytest.log 2>&1
tools/ab_run.sh gpurun_out/r2h_ab.log 2 quant float
