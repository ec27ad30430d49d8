#!/bin/bash
O=gpurun_out; mkdir -p $O
SCV_LIB=variants/lib_nocgp.so timeout 150 python tools/slab_check.py old 500 8 2>&1 | tail -1
timeout 150 python tools/slab_check.py new 500 8 2>&1 | tail -1
python tools/slab_check.py --cmp old new
SCV_LIB=variants/lib_nocgp.so timeout 150 python tools/slab_check.py old2 1016 8 2>&1 | tail -1
timeout 150 python tools/slab_check.py new2 1016 8 2>&1 | tail -1
python tools/slab_check.py --cmp old2 new2
rm -f $O/slab_*.npz
run() { SCV_LIB=$2 timeout 200 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e 2>$O/r02n_$1.err | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$1 ms/map', round(d['ms_per_step'],1), 'rt', d['roundtrip_rel_err']); print({k: round(v,1) for k,v in d['stages_ms_per_step'].items() if v>1})"; }
run base paper_1511_05578_b200/libscurve_b200.so

SCV_LIB=variants/lib_stats.so timeout 200 python tools/pipe_stats.py 32 2>&1 | tail -5; timeout 100 python tools/stagebench.py 2047 | tail -1
