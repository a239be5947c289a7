#!/bin/bash
# build a diagnostics variant of libpsa.so into exp/ (git-ignored, travels to the GPU box):
#   tools/build_variant.sh NAME -DFLAG ...   -> exp/libpsa_NAME.so, load with PSA_LIB_PATH
set -e
cd "$(dirname "$0")/.."
mkdir -p exp
name=$1; shift
C=paper_2412_03594_b200/csrc
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -shared \
  -Xcompiler -fPIC -cudart static -I include "$@" $C/psa_kernel.cu $C/psa_api.cpp $C/psa_plan.cpp \
  $C/psa_prefix.cpp -o exp/libpsa_$name.so
