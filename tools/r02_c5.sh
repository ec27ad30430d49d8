#!/bin/bash
# C5 (L=2048 spin 2, streamed) with the base build and every variants/lib_*.so
run() { SCV_LIB=$2 timeout 600 python bench.py --streamed --L 2048 --spin 2 --jmin 4 --no-cpu-baseline --no-e2e --steps 2 --warmup 1 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$1 ms/map', round(d['ms_per_step'],1), 'rt', d['roundtrip_rel_err'], {k: round(v,1) for k,v in d['stages_ms_per_step'].items() if v>20})"; }
run base paper_1511_05578_b200/libscurve_b200.so
for f in variants/lib_*.so; do v=$(basename $f .so); run ${v#lib_} $f; done
