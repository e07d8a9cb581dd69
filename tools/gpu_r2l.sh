# round 2: full GPU suite + full bench + reference arm (short)
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r2l_pytest.log 2>&1
timeout 1500 python bench.py > gpurun_out/r2l_bench.log 2>&1
