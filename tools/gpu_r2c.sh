# round 2: gpu tests, full bench (sustained), short reference arm
timeout 1500 python -m pytest tests -m gpu -x -q -p no:randomly > gpurun_out/r2c_pytest.log 2>&1
timeout 1200 python bench.py > gpurun_out/r2c_bench.log 2>&1
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r2c_ref.log 2>&1
