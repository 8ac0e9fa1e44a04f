#!/bin/bash
# Experiment builds of the engine with -D switches: scripts/lib_<name>.so
set -e
cd "$(dirname "$0")/.."
build() { name=$1; shift
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared \
    --expt-relaxed-constexpr "$@" -o scripts/lib_$name.so paper_2602_17206_b200/csrc/sdtw_capi.cu -ldl; echo built $name; }
for spec in "$@"; do name=${spec%%:*}; flags=${spec#*:}; build $name $flags & done; wait
