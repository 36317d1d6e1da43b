#!/bin/bash
# A/B experiment builds: profiles/ab_build.sh <name> [extra nvcc flags...]
# -> ab/libpe_<name>.so (git-ignored; run with PE_LIB_OVERRIDE=ab/libpe_<name>.so)
set -e
R=$(cd "$(dirname "$0")/.." && pwd)
name=$1; shift
C=$R/paper_2505_16932_b200/csrc
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared \
  -I $R/include -I $C "$@" $C/pe_api.cu $C/pe_coeffs.cpp $C/pe_dist.cpp -ldl -o $R/ab/libpe_$name.so
