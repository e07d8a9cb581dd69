# round 2: DMMA kernel K-split A/B + parity
for r in 1 2; do for v in mma1 mma2; do echo "== $v" >> gpurun_out/r2p_fp64.log; SPCP_LIB_PATH=ab/lib_$v.so timeout 300 python tools/fp64_probe.py 10 >> gpurun_out/r2p_fp64.log 2>&1; done; done
timeout 1200 python -m pytest tests/test_parity_gpu.py tests/test_scale_gpu.py tests/test_solver_gpu.py tests/test_sddmm_gpu.py -m gpu -q > gpurun_out/r2p_pytest.log 2>&1
