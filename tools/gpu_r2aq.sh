#!/bin/bash
mkdir -p gpurun_out
for t in gold gnew gnew2 gnew2; do echo "== $t" >> gpurun_out/r2aq_gram.txt; SPCP_LIB_PATH=ab/lib_$t.so timeout 300 python tools/gram_bench.py >> gpurun_out/r2aq_gram.txt 2>&1; done
timeout 900 python -m pytest tests/test_solver_gpu.py tests/test_dist_gpu.py tests/test_line_gpu.py -x -q > gpurun_out/r2aq_pytest.log 2>&1
timeout 900 python tools/ttc_trace_probe.py c2 c5 > gpurun_out/r2aq_trace.log 2>&1
echo done
