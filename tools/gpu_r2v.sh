# round 2: certificate starting block 16 vs 8 (C2)
for r in 1 2; do for b in 16 8; do echo "== block $b" >> gpurun_out/r2v_cert.log
  timeout 300 python tools/cert_time_probe.py $b >> gpurun_out/r2v_cert.log 2>&1; done; done
