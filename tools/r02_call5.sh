#!/bin/bash
# r02 GPU pass 5: pipelined column generation -- bench, variants, full-size parity
O=gpurun_out; mkdir -p $O
run() { SCV_LIB=$2 timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e 2>$O/r02e_$1.err | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$1 ms/map', round(d['ms_per_step'],1), 'rt', d['roundtrip_rel_err']); print({k: round(v,1) for k,v in d['stages_ms_per_step'].items() if v>1})"; }
run base paper_1511_05578_b200/libscurve_b200.so
for f in variants/lib_*.so; do v=$(basename $f .so); run ${v#lib_} $f; done
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_full.py -m gpu -x -q -k "1024 or full_size or c4 or slab" > $O/r02e_pytest.log 2>&1; tail -5 $O/r02e_pytest.log
