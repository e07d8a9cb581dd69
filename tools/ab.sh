#!/bin/bash
# A/B kernel_ms of compile-time variants: VARIANTS="name:flags;name:flags"
cd ${GRAFT_REPO_ROOT:-.}
O=gpurun_out; mkdir -p $O; L=$O/ab_${TAG:-x}.log; rm -f $L
IFS=';' read -ra VS <<< "$VARIANTS"
for v in "${VS[@]}"; do
  name=${v%%:*}; flags=${v#*:}
  make -B EXTRA="$flags" > $O/ab_make.log 2>&1 || { echo "$name build failed" >> $L; continue; }
  for env in ${ENVS:-X=1}; do
    echo "$name $env $(env $env timeout 120 python bench.py --steps 50 --warmup 3 --skip-cpu --skip-e2e --skip-ttc 2>&1 | grep -o '"ms_per_step": [0-9.]*\|"kernel_ms": [0-9.]*' | tr '\n' ' ')" >> $L
  done
done
make -B > /dev/null 2>&1
