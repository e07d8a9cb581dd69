# round 2: chunk picking for the (band x chunk) grids: fp64 evaluation + certificate A/B
for r in 1 2; do for v in head chunks; do echo "== $v" >> gpurun_out/r2r_ab.log
  SPCP_LIB_PATH=ab/lib_$v.so timeout 300 python tools/fp64_probe.py 10 >> gpurun_out/r2r_ab.log 2>&1
  SPCP_LIB_PATH=ab/lib_$v.so timeout 300 python tools/cert_time_probe.py >> gpurun_out/r2r_ab.log 2>&1
done; done
