#!/bin/bash
# round 2af: epilogue instruction-count sensitivity (extra FFMA2 per element pair)
mkdir -p gpurun_out
tools/ab_run.sh gpurun_out/r2ag_ab.txt 3 p0 p1 p2
echo done
