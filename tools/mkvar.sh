#!/bin/bash
# Build a launch-shape variant of the library into variants/lib_NAME.so.
# usage: tools/mkvar.sh NAME ROW2047 COL2047 ROW1023 COL1023 [-DMACRO=V ...]   (each R_NT_MINB, "-" keeps the default)
name=$1; shift
cd "$(dirname "$0")/.."
f=paper_1511_05578_b200/csrc/pfa.cu
cp $f /tmp/pfa_backup_$$.cu
i=0
for key in ROW2047 COL2047 ROW1023 COL1023; do
  i=$((i+1)); v=${!i}
  if [ -n "$v" ] && [ "$v" != "-" ]; then
    sed -i -E "s/^#define SCV_${key} .*/#define SCV_${key} ${v//_/, }/" $f
  fi
done
shift 4 2>/dev/null
python -m paper_1511_05578_b200.build --force --out=$PWD/variants/lib_$name.so "$@" | tail -1
cp /tmp/pfa_backup_$$.cu $f
rm -f /tmp/pfa_backup_$$.cu
