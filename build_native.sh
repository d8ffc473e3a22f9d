#!/usr/bin/env bash
# Build libhapod_b200.so in-tree for sm_100a (no GPU needed: nvcc cross-compiles).
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
SRC="$HERE/paper_1607_05210_b200/csrc"
OUT="$HERE/paper_1607_05210_b200/libhapod_b200.so"
OBJ="$HERE/build/obj"
NVCC="${NVCC:-nvcc}"
mkdir -p "$OBJ"
FLAGS=(-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC
       -Xptxas -warn-spills -I"$HERE/include")
pids=()
for f in hp_gemm hp_jacobi hp_podops hp_pstrf hp_tridiag hp_capi; do
  "$NVCC" "${FLAGS[@]}" -c "$SRC/$f.cu" -o "$OBJ/$f.o" &
  pids+=($!)
done
for p in "${pids[@]}"; do wait "$p"; done
"$NVCC" -gencode arch=compute_100a,code=sm_100a -shared "$OBJ"/*.o -o "$OUT.tmp"
mv "$OUT.tmp" "$OUT"
echo "built $OUT"
