#!/bin/bash
# quick A/B: bench (2 steps) of the base build and every variants/lib_*.so except lib_stats/lib_old
O=gpurun_out; mkdir -p $O; TAG=${1:-r02q}
run() { SCV_LIB=$2 timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e $3 2>$O/${TAG}_$1.err | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$1 ms/map', round(d['ms_per_step'],1), 'rt', d['roundtrip_rel_err']); print({k: round(v,1) for k,v in d['stages_ms_per_step'].items() if v>1})"; }
run base paper_1511_05578_b200/libscurve_b200.so
for f in variants/lib_*.so; do v=$(basename $f .so); [ $v = lib_stats ] || [ $v = lib_old ] || run ${v#lib_} $f; done
