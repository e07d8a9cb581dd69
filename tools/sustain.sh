#!/bin/bash
# kernel_ms vs timed-region length (power/thermal sensitivity of the on-chip-bound kernel)
cd ${GRAFT_REPO_ROOT:-.}; O=gpurun_out; mkdir -p $O; L=$O/sustain.log; rm -f $L
for s in 20 50 200 1000 200 50; do
  echo "steps $s $(timeout 300 python bench.py --steps $s --warmup 3 --skip-cpu --skip-e2e --skip-ttc 2>&1 | grep -o '"ms_per_step": [0-9.]*\|"kernel_ms": [0-9.]*\|"sm_mhz": [0-9.]*\|"sm_mhz_min": [0-9.]*\|"reasons": \[[^]]*\]' | tr '\n' ' ')" >> $L
done
nvidia-smi -q -d POWER,TEMPERATURE,CLOCK | grep -E "Power Draw|Limit|Temp|Clocks|SM |Memory " | head -30 >> $L
