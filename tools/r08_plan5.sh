#!/bin/bash
# A/B of the K = 4095 plans on the C5 streamed map
O=gpurun_out; mkdir -p $O
for lib in paper_1511_05578_b200/libscurve_b200.so variants/lib_*.so; do
  [ -f $lib ] || continue
  SCV_LIB=$lib timeout 600 python bench.py --streamed --L 2048 --spin 2 --jmin 4 --no-cpu-baseline --no-e2e --steps 2 --warmup 1 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$lib', d['config']['L'], 'ms/map', round(d['ms_per_step'],1), 'rt', d['roundtrip_rel_err'], {k: round(v,1) for k,v in d['stages_ms_per_step'].items() if v>20})"
done
