# round 2: coalesced sparse-observation passes; sanitizers
timeout 900 python -m pytest tests/test_sddmm_gpu.py -q > gpurun_out/r2j_sddmm.log 2>&1
timeout 1200 python tools/sddmm_probe.py > gpurun_out/r2j_sddmm_probe.log 2>&1
timeout 900 compute-sanitizer --tool memcheck python tools/sanitize_probe.py > gpurun_out/r2j_memcheck.log 2>&1
timeout 900 compute-sanitizer --tool racecheck python tools/sanitize_probe.py > gpurun_out/r2j_racecheck.log 2>&1
timeout 900 compute-sanitizer --tool synccheck python tools/sanitize_probe.py > gpurun_out/r2j_synccheck.log 2>&1
