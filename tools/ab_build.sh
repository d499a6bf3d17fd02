#!/bin/bash
# tools/ab_build.sh NAME [extra nvcc flags] -- build libcoat.so from the current
# sources into build_ab/NAME/ (for COAT_LIB=build_ab/NAME/libcoat.so A/B runs).
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
NAME=$1; shift
OUT=$ROOT/build_ab/$NAME
mkdir -p $OUT/obj
ARCH="-gencode arch=compute_100a,code=sm_100a"
FLAGS="-O3 -std=c++17 $ARCH -lineinfo --fmad=false -prec-div=true -prec-sqrt=true -ftz=false -Xcompiler -fPIC -Xcompiler -ffp-contract=off -I$ROOT/include $*"
pids=()
for f in $ROOT/paper_2410_19313_b200/csrc/*.cu; do
  nvcc $FLAGS -c -o $OUT/obj/$(basename $f .cu).o $f &
  pids+=($!)
done
for p in "${pids[@]}"; do wait $p || { echo "compile failed"; exit 1; }; done
nvcc $ARCH -shared -o $OUT/libcoat.so $OUT/obj/*.o -lcudart
rm -rf $OUT/obj
echo built $OUT/libcoat.so
