# round 2: G^T U gh/gl fold in the drain; fp64 dispatch split; subspace block growth
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r2e_pytest.log 2>&1
timeout 900 python bench.py --skip-cpu > gpurun_out/r2e_bench.log 2>&1
timeout 300 python tools/fp64_probe.py 10 > gpurun_out/r2e_fp64.log 2>&1
