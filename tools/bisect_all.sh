#!/bin/bash
# Full bisection of the fused TC kernel (box-side): runtime switches
# (SPCP_TC_DEBUG) x compile-time variants (SPCP_TC_BISECT_*), kernel_ms each.
cd ${GRAFT_REPO_ROOT:-.}
O=gpurun_out; mkdir -p $O; L=$O/bisall_${TAG:-x}.log; rm -f $L
for v in ${VARIANTS:-NONE SPCP_TC_BISECT_EPI_SKIP SPCP_TC_BISECT_NO_SMEM SPCP_TC_BISECT_NO_TMA}; do
  make -B EXTRA="-D$v $XEXTRA" > /dev/null 2>&1 || { echo "$v build failed" >> $L; continue; }
  for d in ${DEBUGS:-0 8 16 32 64 3 11}; do
    echo "$v debug=$d $(SPCP_TC_DEBUG=$d timeout 120 python bench.py --steps 50 --warmup 3 --skip-cpu --skip-e2e --skip-ttc 2>&1 | grep -o '"kernel_ms": [0-9.]*')" >> $L
  done
done
make -B > /dev/null 2>&1
