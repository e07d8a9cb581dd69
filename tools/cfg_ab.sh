#!/bin/bash
# configs_probe under two builds on the same box
cd ${GRAFT_REPO_ROOT:-.}; O=gpurun_out; mkdir -p $O; rm -f $O/cfg_ab.log
for v in "lpi2:-DSPCP_REDUCE_FORCE_LPI2" "skew:" "lpi2b:-DSPCP_REDUCE_FORCE_LPI2" "skewb:"; do
  name=${v%%:*}; flags=${v#*:}
  make -B EXTRA="$flags" > /dev/null 2>&1
  echo "== $name" >> $O/cfg_ab.log
  timeout 300 python tools/configs_probe.py >> $O/cfg_ab.log 2>&1
done
make -B > /dev/null 2>&1
