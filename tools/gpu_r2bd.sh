#!/bin/bash
# round 2bd: G.V on an early TMEM barrier ring (aliasing-safe): smoke first
# with a short timeout, then A/B + parity
mkdir -p gpurun_out
SPCP_LIB_PATH=ab/lib_e1.so timeout 120 python bench.py --steps 20 --warmup 3 --skip-cpu --skip-e2e --skip-ttc --skip-c5 > gpurun_out/r2bd_probe.log 2>&1
echo "probe rc=$?" >> gpurun_out/r2bd_probe.log
if grep -q "probe rc=0" gpurun_out/r2bd_probe.log; then
  for r in 1 2 3; do for t in e0 e1; do
    echo "$t round $r: $(SPCP_LIB_PATH=ab/lib_$t.so timeout 120 python bench.py --steps 200 --warmup 3 --skip-cpu --skip-e2e --skip-ttc --skip-c5 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']
print(f\"step {d['ms_per_step']:.4f} kernel {r['kernel_ms']:.4f} burst_kernel {r['burst']['kernel_ms']:.4f}\")" 2>&1 | tail -1)" >> gpurun_out/r2bd_ab.txt
  done; done
  for t in e0 e1; do echo "== $t configs" >> gpurun_out/r2bd_ab.txt; SPCP_LIB_PATH=ab/lib_$t.so timeout 300 python tools/configs_probe.py >> gpurun_out/r2bd_ab.txt 2>&1; done
  SPCP_LIB_PATH=ab/lib_e1.so timeout 600 python -m pytest tests/test_parity_gpu.py tests/test_configs_gpu.py -x -q > gpurun_out/r2bd_pytest.log 2>&1
fi
echo done
