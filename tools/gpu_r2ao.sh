#!/bin/bash
# round 2ao: fold kernel without the local-memory s[] (and register-capped variants)
mkdir -p gpurun_out
tools/ab_run.sh gpurun_out/r2ao_ab.txt 3 old new new4 new3
echo done
