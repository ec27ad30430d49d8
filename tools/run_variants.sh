#!/bin/bash
# On the GPU box: fftbench + a short L=1024 bench for every variants/lib_*.so.
# usage: tools/run_variants.sh [K-list] [bench-args...]
KS=${1:-1023,2047}; shift
for f in variants/lib_*.so; do
  v=$(basename $f .so); v=${v#lib_}
  echo "== $v"
  [ "$KS" != none ] && SCV_LIB=$f timeout 180 python tools/fftbench.py $KS 2>&1 | grep "K="
  SCV_LIB=$f timeout 400 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e "$@" 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench ms/map', round(d['ms_per_step'],1), 'rt', '%.1e' % d['roundtrip_rel_err'], {k: round(v,1) for k, v in d['stages_ms_per_step'].items() if v > 20})"
done
