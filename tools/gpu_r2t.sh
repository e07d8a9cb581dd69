# round 2: per-block maxima instead of same-address atomics: A/B + tests
tools/ab_run.sh gpurun_out/r2t_ab.log 2 atom bmax
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r2t_pytest.log 2>&1
