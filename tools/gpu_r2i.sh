# round 2: sparse-observation path: tests, crossover probe; full test suite
timeout 900 python -m pytest tests/test_sddmm_gpu.py -q -s > gpurun_out/r2i_sddmm.log 2>&1
timeout 1200 python tools/sddmm_probe.py > gpurun_out/r2i_sddmm_probe.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r2i_pytest.log 2>&1
