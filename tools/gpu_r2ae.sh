#!/bin/bash
# round 2ae: GPU suite + bench line after the line-search / sketch work
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r2ae_pytest.log 2>&1
timeout 1500 python bench.py > gpurun_out/r2ae_bench.log 2>&1
echo done
