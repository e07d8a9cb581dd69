# round 2: segment fold kernel vs the LPI reduce: A/B + tests
tools/ab_run.sh gpurun_out/r2s_ab.log 2 lpi fold
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r2s_pytest.log 2>&1
