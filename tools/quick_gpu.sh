#!/bin/bash
# quick GPU iteration: numerics check, GPU tests, a short bench line
cd ${GRAFT_REPO_ROOT:-.}
O=gpurun_out; mkdir -p $O
timeout 300 python tools/tc_check.py > $O/q_tc_check.log 2>&1; echo "rc $?" >> $O/q_tc_check.log
timeout 120 python bench.py --steps 50 --warmup 3 --skip-cpu --skip-e2e --skip-ttc > $O/q_bench.log 2>&1; echo "rc $?" >> $O/q_bench.log
SPCP_TC_LAYOUT=split timeout 120 python bench.py --steps 50 --warmup 3 --skip-cpu --skip-e2e --skip-ttc > $O/q_bench_split.log 2>&1
[ -n "$TESTS" ] && { timeout 600 python -m pytest tests -m gpu -x -q > $O/q_pytest.log 2>&1; echo "rc $?" >> $O/q_pytest.log; }
exit 0
