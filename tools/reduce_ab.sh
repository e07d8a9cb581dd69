#!/bin/bash
# reduce-kernel variants: cold ncu launch time + warm bench step
cd ${GRAFT_REPO_ROOT:-.}; O=gpurun_out; mkdir -p $O; L=$O/reduce_ab.log; rm -f $L
for lpi in ${LPIS:-4 8 16}; do
  make -B EXTRA="-DSPCP_REDUCE_LPI=$lpi" > /dev/null 2>&1 || { echo "lpi $lpi build failed" >> $L; continue; }
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"tc_reduce" -c 6 --csv --log-file $O/ra_$lpi.csv python bench.py --steps 3 --warmup 3 --skip-cpu --skip-e2e --skip-ttc > /dev/null 2>&1
  echo "lpi $lpi cold_us $(grep tc_reduce $O/ra_$lpi.csv | tail -3 | awk -F'","' '{print $NF}' | tr -d '"' | tr '\n' ' ') $(timeout 120 python bench.py --steps 200 --warmup 3 --skip-cpu --skip-e2e --skip-ttc 2>&1 | grep -o '"ms_per_step": [0-9.]*\|"kernel_ms": [0-9.]*' | tr '\n' ' ')" >> $L
done
make -B > /dev/null 2>&1
