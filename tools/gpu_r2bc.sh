#!/bin/bash
# round 2bc: final build sanity: GPU suite + smoke + a short bench
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r2bc_pytest.log 2>&1
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r2bc_smoke.log 2>&1
timeout 900 python bench.py --steps 50 --warmup 5 --skip-ttc --skip-c5 --skip-cpu > gpurun_out/r2bc_bench.log 2>&1
echo done
