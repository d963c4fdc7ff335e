#!/bin/bash
# Build an experimental libdooly variant: tools/build_variant.sh NAME FILE.cu "-DMACRO=VAL ..."
# recompiles FILE.cu with the extra flags against the normal objects and links
# tools/_build/libdooly_NAME.so (load it with DOOLY_LIB_PATH=...).
set -e
cd "$(dirname "$0")/../paper_2605_07985_b200/csrc"
make -s >/dev/null
NAME=$1; FILE=$2; EXTRA=$3
OBJ=../../build/obj
VOBJ=../../build/obj_$NAME
rm -rf "$VOBJ"; cp -r "$OBJ" "$VOBJ"
ARCH="-gencode arch=compute_100a,code=sm_100a"
/usr/local/cuda/bin/nvcc -O3 -std=c++17 $ARCH -lineinfo -Xcompiler -fPIC,-O3 -Xptxas -v --cudart static \
  $EXTRA -dc -o "$VOBJ/${FILE%.cu}.o" "$FILE" 2> "$VOBJ/${FILE%.cu}.ptxas.txt"
mkdir -p ../../tools/_build
/usr/local/cuda/bin/nvcc $ARCH -shared --cudart static -o ../../tools/_build/libdooly_$NAME.so "$VOBJ"/*.o -lnccl
grep -A1 "sha256_records" "$VOBJ/${FILE%.cu}.ptxas.txt" | grep -o "Used [0-9]* registers" | head -2 || true
