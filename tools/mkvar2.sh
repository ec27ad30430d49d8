#!/bin/bash
# Build a variant library variants/lib_NAME.so with pfa.cu macro overrides.
# usage: tools/mkvar2.sh NAME KEY=V_V_V ...   (rewrites "#define SCV_KEY ..." in pfa.cu, '_' -> ', ')
name=$1; shift
cd "$(dirname "$0")/.."
f=paper_1511_05578_b200/csrc/pfa.cu
cp $f /tmp/pfa_backup_$$.cu
for kv in "$@"; do
  key=${kv%%=*}; v=${kv#*=}
  grep -q "^#define SCV_${key} " $f || { echo "no macro SCV_${key}"; cp /tmp/pfa_backup_$$.cu $f; exit 1; }
  sed -i -E "s/^#define SCV_${key} .*/#define SCV_${key} ${v//_/, }/" $f
done
mkdir -p variants
python -m paper_1511_05578_b200.build --force --out=$PWD/variants/lib_$name.so | tail -1
cp /tmp/pfa_backup_$$.cu $f
rm -f /tmp/pfa_backup_$$.cu
