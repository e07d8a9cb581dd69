#!/bin/bash
# Compile-time bisection variants of the fused TC kernel (box-side): each
# variant is rebuilt and timed (kernel_ms), with and without the MMAs.
cd ${GRAFT_REPO_ROOT:-.}
O=gpurun_out; mkdir -p $O; rm -f $O/bisv.log
for v in ${VARIANTS:-NONE SPCP_TC_BISECT_EPI_SKIP SPCP_TC_BISECT_NO_SMEM SPCP_TC_BISECT_NO_TMA}; do
  make -B EXTRA=-D$v > /dev/null 2>&1 || { echo "$v build failed" >> $O/bisv.log; continue; }
  for d in 0 8 3; do
    echo "$v debug=$d $(SPCP_TC_DEBUG=$d timeout 120 python bench.py --steps 20 --warmup 3 --skip-cpu --skip-e2e --skip-ttc 2>&1 | grep -o '"kernel_ms": [0-9.]*')" >> $O/bisv.log
  done
done
