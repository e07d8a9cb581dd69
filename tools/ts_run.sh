#!/bin/bash
# Timestamp builds (CTA 0, first 64 tiles) of the fused TC kernel for a list of
# SPCP_TC_DEBUG values and compile variants; raw tables land in gpurun_out/.
cd ${GRAFT_REPO_ROOT:-.}
O=gpurun_out; mkdir -p $O
for v in ${VARIANTS:-NONE}; do
  make -B EXTRA="-DSPCP_TC_TIMESTAMPS -D$v $XEXTRA" > $O/ts_make.log 2>&1 || { echo "$v build failed"; continue; }
  for d in ${DEBUGS:-4 12}; do
    SPCP_TC_DEBUG=$d timeout 120 python bench.py --steps 3 --warmup 3 --skip-cpu --skip-e2e --skip-ttc > /dev/null 2>&1
    cp -f $O/tc_ts.txt $O/ts_${TAG:-x}_${v}_$d.txt
  done
done
make -B > /dev/null 2>&1
