#!/bin/bash
# Build a kernel variant library: scripts/build_variant.sh NAME [-DFLAG=V ...]
# -> paper_2506_03065_b200/variants/NAME.so (select with SVD_LIB=<path>)
set -e
cd "$(dirname "$0")/.."
name=$1; shift
mkdir -p paper_2506_03065_b200/variants
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC \
  -Xcompiler -fvisibility=default -shared -I include "$@" \
  paper_2506_03065_b200/csrc/svd_plan.cpp paper_2506_03065_b200/csrc/svd_attn_fwd.cu paper_2506_03065_b200/csrc/svd_layer.cu \
  paper_2506_03065_b200/csrc/svd_key_mass.cu paper_2506_03065_b200/csrc/svd_gemm.cu \
  -o paper_2506_03065_b200/variants/$name.so
