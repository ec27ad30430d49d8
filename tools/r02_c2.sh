#!/bin/bash
# ring kernels at K = 511: parity at L = 256, then L = 256 and C4 benches of the base build and variants
timeout 900 python -m pytest tests/test_gpu_parity_full.py tests/test_gpu_parity.py -m gpu -x -q -k "256 or quadrature or slab or linear" 2>&1 | tail -2
run() { SCV_LIB=$2 timeout 300 python bench.py --steps $4 --warmup 3 --no-cpu-baseline --no-e2e $3 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$1 ms/map', round(d['ms_per_step'],2), 'rt', d['roundtrip_rel_err'], {k: round(v,2) for k,v in d['stages_ms_per_step'].items() if v>0.2})"; }
for f in paper_1511_05578_b200/libscurve_b200.so variants/lib_*.so; do v=$(basename $f .so); run L256_$v $f "--L 256 --jmin 2" 20; run C4_$v $f "" 2; done
