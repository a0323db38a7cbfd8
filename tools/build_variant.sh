#!/bin/bash
# A/B kernel experiments: build libbornsweep.so with extra -D flags into variants/<name>/
#   tools/build_variant.sh <name> "-DBS_ROW_SMEM=0 ..." [TU ...]
# With TU names (e.g. sweep_L9 bornsweep) only those are recompiled; the other objects are
# taken from the main build (paper_2603_18527_b200/csrc/obj).  Load the result with
# BP_LIB_PATH=variants/<name>/libbornsweep.so (tools/kbench.py, bench.py).
set -e
NAME=$1; shift
FLAGS="$1"; shift || true
ROOT=$(cd "$(dirname "$0")/.." && pwd)
SRC=$ROOT/paper_2603_18527_b200/csrc
OUT=$ROOT/variants/$NAME
mkdir -p $OUT/obj
NV="/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -ccbin /usr/bin/g++ --diag-suppress 128 -I$ROOT/include -I$SRC $FLAGS"
if [ $# -gt 0 ]; then
  cp $SRC/obj/*.o $OUT/obj/
  for tu in "$@"; do echo $tu; done | xargs -P 12 -I{} sh -c "$NV -c -o $OUT/obj/{}.o $SRC/{}.cu"
else
  ls $SRC/*.cu | xargs -P 12 -I{} sh -c "$NV -c -o $OUT/obj/\$(basename {} .cu).o {}"
fi
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -ccbin /usr/bin/g++ -o $OUT/libbornsweep.so $OUT/obj/*.o
echo built $OUT/libbornsweep.so
