#!/bin/bash
mkdir -p gpurun_out
timeout 600 python tools/init_probe.py > gpurun_out/r2y_init.log 2>&1
echo done
