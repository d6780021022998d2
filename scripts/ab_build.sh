#!/bin/bash
# Build a variant of the library with extra nvcc defines for A/B timing:
#   scripts/ab_build.sh <name> -DFOO=1 ...  ->  build/ab/<name>/libcrvpinn.so  (use via CRVPINN_LIB)
set -e
NAME=$1; shift
ROOT=$(cd "$(dirname "$0")/.." && pwd)
OUT=$ROOT/build/ab/$NAME
mkdir -p $OUT
NV=/usr/local/cuda/bin/nvcc
FL="-gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC --expt-relaxed-constexpr"
pids=()
for src in $ROOT/paper_2604_20731_b200/csrc/*.cu; do
  $NV $FL "$@" -c $src -o $OUT/$(basename ${src%.cu}).o & pids+=($!)
done
for p in ${pids[@]}; do wait $p; done
$NV -gencode arch=compute_100a,code=sm_100a -shared -cudart shared -Xlinker -rpath,/usr/local/cuda/lib64 -o $OUT/libcrvpinn.so $OUT/*.o
echo $OUT/libcrvpinn.so
