#!/bin/bash
# Same-box A/B of library variants: interleaved bench / config-probe runs.
#   tools/ab_run.sh OUT ROUNDS TAG... (libraries ab/lib_TAG.so)
out=$1; rounds=$2; shift 2
for r in $(seq 1 $rounds); do
  for tag in "$@"; do
    res=$(SPCP_LIB_PATH=ab/lib_$tag.so timeout 300 python bench.py --steps 200 --warmup 3 \
          --skip-cpu --skip-e2e --skip-ttc --skip-c5 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']
print(f\"step {d['ms_per_step']:.4f} kernel {r['kernel_ms']:.4f} frac {r['frac']:.3f} burst_kernel {r['burst']['kernel_ms']:.4f} mhz {d['clocks']['sm_mhz']}\")" 2>&1)
    echo "$tag round $r: $res" >> $out
  done
done
for tag in "$@"; do
  echo "== $tag configs" >> $out
  SPCP_LIB_PATH=ab/lib_$tag.so timeout 600 python tools/configs_probe.py >> $out 2>&1
done
