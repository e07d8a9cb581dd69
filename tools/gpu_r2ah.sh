#!/bin/bash
# round 2ah: epilogue instruction trims (FHFMA lo piece, XOR-swizzled shared addresses)
mkdir -p gpurun_out
tools/ab_run.sh gpurun_out/r2ah_ab.txt 3 base fh fx
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_configs_gpu.py tests/test_sddmm_gpu.py -x -q > gpurun_out/r2ah_pytest.log 2>&1
echo done
