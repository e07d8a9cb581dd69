#!/bin/bash
mkdir -p gpurun_out
for t in gold gnew gold gnew; do echo "== $t" >> gpurun_out/r2ap_gram.txt; SPCP_LIB_PATH=ab/lib_$t.so timeout 300 python tools/gram_bench.py >> gpurun_out/r2ap_gram.txt 2>&1; done
timeout 900 python -m pytest tests/test_solver_gpu.py tests/test_dist_gpu.py -x -q > gpurun_out/r2ap_pytest.log 2>&1
echo done
