#!/bin/bash
# Variant of the library with extra nvcc defines on mlp_tc.cu only (the other objects come from the
# default build in paper_2604_20731_b200/build_obj): scripts/ab_build_tc.sh <name> -DFOO=1 ... -> build/ab/<name>/libcrvpinn.so
set -e
NAME=$1; shift
ROOT=$(cd "$(dirname "$0")/.." && pwd)
OUT=$ROOT/build/ab/$NAME
OBJ=$ROOT/paper_2604_20731_b200/build_obj
mkdir -p $OUT
NV=/usr/local/cuda/bin/nvcc
FL="-gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC --expt-relaxed-constexpr"
$NV $FL "$@" -c $ROOT/paper_2604_20731_b200/csrc/mlp_tc.cu -o $OUT/mlp_tc.o
$NV -gencode arch=compute_100a,code=sm_100a -shared -cudart shared -Xlinker -rpath,/usr/local/cuda/lib64 -o $OUT/libcrvpinn.so \
  $OUT/mlp_tc.o $OBJ/crvpinn.o $OBJ/fields.o $OBJ/gram.o $OBJ/iga.o $OBJ/mlp_simt.o
echo $OUT/libcrvpinn.so
