#!/bin/sh
# Build libmeshreg_b200.so for sm_100a (in-tree, next to the Python package).
# Host setup code is compiled with -ffp-contract=off: its fp64 geometry must
# round exactly like numpy (bit-exact CSR / coefficients / orientation).
set -e
HERE=$(cd "$(dirname "$0")" && pwd)
OUT=${1:-$HERE/../libmeshreg_b200.so}
NVCC=${NVCC:-nvcc}
$NVCC -std=c++17 -O3 -lineinfo -gencode arch=compute_100a,code=sm_100a $MRB_NVCC_FLAGS \
  -Xcompiler -fPIC,-ffp-contract=off -Xptxas -v -shared \
  -I"$HERE/../../include" \
  "$HERE/meshreg_b200.cu" "$HERE/mesh_host.cpp" "$HERE/mesher_host.cpp" -o "$OUT.tmp" 2> "$HERE/../../build_ptxas.log" || {
    grep -v "^ptxas info\|^    [0-9]* bytes stack" "$HERE/../../build_ptxas.log" | head -40; exit 1; }
mv "$OUT.tmp" "$OUT"
echo "built $OUT"
