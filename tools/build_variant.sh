#!/bin/bash
# Build an A/B variant of libpoba with extra nvcc flags into libab/<name>/libpoba.so
# (git-ignored; travels to the GPU box).  Use it with POBA_LIB=libab/<name>/libpoba.so.
#   bash tools/build_variant.sh <name> "<extra nvcc flags>"
set -e
NAME=$1; shift
EXTRA="$*"
ROOT=$(cd "$(dirname "$0")/.." && pwd)
OUT=$ROOT/libab/$NAME
OBJ=/tmp/libab_obj/$NAME
mkdir -p "$OUT" "$OBJ"
NVCC=/usr/local/cuda/bin/nvcc
ARCH="-gencode arch=compute_100a,code=sm_100a"
FLAGS="-I $ROOT/include $ARCH -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr $EXTRA"
SRC=${POBA_SRC:-$ROOT/paper_2204_12834_b200/csrc}
pids=()
for f in "$SRC"/*.cu; do
  $NVCC $FLAGS -c "$f" -o "$OBJ/$(basename "$f" .cu).o" & pids+=($!)
done
for f in "$SRC"/*.cpp; do
  g++ -O3 -std=c++17 -fPIC -c "$f" -o "$OBJ/$(basename "$f" .cpp).o" & pids+=($!)
done
for p in "${pids[@]}"; do wait "$p"; done
$NVCC $ARCH -shared -o "$OUT/libpoba.so" "$OBJ"/*.o -lcudart -ldl
echo "$OUT/libpoba.so"
