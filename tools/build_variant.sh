#!/bin/bash
# Build an A/B variant of the library: tools/build_variant.sh <name> <extra nvcc flags...>
# Output: paper_2604_11659_b200/lib/variants/<name>.so (select with HS_LIB_PATH).
set -e
NAME=$1; shift
ROOT=$(cd "$(dirname "$0")/.." && pwd)
SRC=$ROOT/paper_2604_11659_b200/csrc
OUT=$ROOT/paper_2604_11659_b200/lib/variants/$NAME
mkdir -p "$OUT"
FL="-O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC,-O2 --expt-relaxed-constexpr $*"
for f in ops capi runner keygen decode probe; do nvcc $FL -c $SRC/$f.cu -o $OUT/$f.o & done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o "$OUT.so" $OUT/*.o -lcudart
echo "$OUT.so"
