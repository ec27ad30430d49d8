#!/bin/bash
# Build variants/lib_NAME.so with -D macro overrides (all SCV_* knobs are #ifndef-guarded).
# usage: tools/mkvar3.sh NAME -DSCV_X=1 -DSCV_ROWS_GRP=5,96 ...
name=$1; shift
cd "$(dirname "$0")/.."
mkdir -p variants
python -m paper_1511_05578_b200.build --out=$PWD/variants/lib_$name.so "$@" 2>&1 | tail -2
# the variant's objects are not needed once it is linked (build/ travels with gpurun snapshots)
rm -rf build/obj/var_lib_$name
