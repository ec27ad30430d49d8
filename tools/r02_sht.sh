#!/bin/bash
# SHT contraction variants: parity tests on the base build, then the stage time of each build (C4 bench, 2 steps)
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "sht or halfpi or config1 or transform_golden or transform_vs_oracle" 2>&1 | tail -2
run() { SCV_LIB=$2 timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$1 ms/map', round(d['ms_per_step'],1), 'rt', d['roundtrip_rel_err'], {k: round(v,2) for k,v in d['stages_ms_per_step'].items() if k.startswith('sht') or k=='beta_sht'})"; }
run base paper_1511_05578_b200/libscurve_b200.so
for f in variants/lib_*.so; do v=$(basename $f .so); run ${v#lib_} $f; done
