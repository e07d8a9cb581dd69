#!/bin/bash
# round 2ay: four S buffers (two G^T U accumulators) with G.V first (A/B)
mkdir -p gpurun_out
tools/ab_run.sh gpurun_out/r2ay_ab.txt 3 n3 n4
echo done
