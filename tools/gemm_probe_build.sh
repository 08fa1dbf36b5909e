#!/bin/bash
# build tools/gemm_mn_probe from a copy of gemm.cu with the phase trace compiled in
#   tools/gemm_probe_build.sh [out-name [extra sed expression]]
set -e
cd "$(dirname "$0")/.."
OUT=${1:-gemm_mn_probe}
mkdir -p build_probe/$OUT
sed -e 's/constexpr bool kGemmTrace = false;/constexpr bool kGemmTrace = true;/' ${2:+-e "$2"} \
  paper_1710_06952_b200/csrc/gemm.cu > build_probe/$OUT/gemm_traced.cu
nvcc -O2 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I include -I paper_1710_06952_b200/csrc -I build_probe/$OUT \
  tools/gemm_mn_probe.cu -o build_probe/$OUT/probe -lcuda
