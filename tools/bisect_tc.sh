#!/bin/bash
# Pipeline bisection of the fused TC kernel on the box: kernel time with the
# MMAs / partial stores switched off, then a timestamp build (CTA 0, per tile).
cd ${GRAFT_REPO_ROOT:-.}
O=gpurun_out; mkdir -p $O; rm -f $O/bis.log
for d in ${BIS_DEBUGS:-0 8 3 11}; do
  echo "debug=$d $(SPCP_TC_DEBUG=$d timeout 300 python bench.py --steps 20 --warmup 3 --skip-cpu --skip-e2e --skip-ttc 2>&1 | grep -o '"kernel_ms": [0-9.]*')" >> $O/bis.log
done
make -B EXTRA=-DSPCP_TC_TIMESTAMPS > $O/bis_make.log 2>&1
for d in 4 12; do
SPCP_TC_DEBUG=$d timeout 300 python bench.py --steps 3 --warmup 3 --skip-cpu --skip-e2e --skip-ttc > /dev/null 2>&1
cp -f $O/tc_ts.txt $O/bis_ts$d.txt
done
