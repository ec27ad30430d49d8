#!/bin/bash
# A/B of the K = 1023 plans: C3 and C4 bench lines per library
O=gpurun_out; mkdir -p $O
for lib in paper_1511_05578_b200/libscurve_b200.so variants/lib_*.so; do
  [ -f $lib ] || continue
  for cfg in "--L 512 --jmin 2 --steps 5" "--steps 2"; do
    SCV_LIB=$lib timeout 300 python bench.py $cfg --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$lib', d['config']['L'], 'ms/map', round(d['ms_per_step'],2), 'rt', d['roundtrip_rel_err'], {k: round(v,2) for k,v in d['stages_ms_per_step'].items() if v>1})"
  done
done
