#!/bin/bash
mkdir -p gpurun_out
timeout 900 python tools/cert_c5_probe.py c2 > gpurun_out/r2al_cert_c2.log 2>&1
echo done
