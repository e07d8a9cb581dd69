#!/bin/bash
# Build variants of libspcp_b200.so for same-box A/B timing (tools/ab_run.sh):
#   tools/ab_build.sh TAG "-DMACRO=VALUE ..." [TAG "..."]...
set -e
cd "$(dirname "$0")/.."
mkdir -p ab
while [ $# -ge 2 ]; do
  tag=$1; flags=$2; shift 2
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared \
    --expt-relaxed-constexpr $flags -o ab/lib_$tag.so paper_1702_02241_b200/csrc/spcp_api.cu &
done
wait
ls -la ab/
