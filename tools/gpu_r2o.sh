# round 2: ncu of the DMMA fp64 evaluation kernel at C2 (k=20)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:f64_mma_kernel -s 2 -c 1 \
  -o gpurun_out/r2o_f64mma python tools/fp64_probe.py 3 > gpurun_out/r2o_ncu.log 2>&1
