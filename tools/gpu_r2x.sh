#!/bin/bash
# round 2x: evaluation trace of the C2 and C5 time to certificate
mkdir -p gpurun_out
timeout 900 python tools/ttc_trace_probe.py c2 c5 > gpurun_out/r2x_trace.log 2>&1
echo done
