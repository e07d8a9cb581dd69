# round 2: KC layout for k <= 32 + G^T U fold: tests, then same-box A/B
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2f_pytest.log 2>&1
tools/ab_run.sh gpurun_out/r2f_ab.log 2 base fold0 fold1
