#!/bin/bash
# r02 GPU pass: A/B of library variants (variants/lib_*.so) against the base build
# usage: tools/r02_variants.sh TAG   (lib_old.so = reference for the slab digests, lib_stats.so = pipeline counters)
O=gpurun_out; mkdir -p $O
TAG=${1:-r02m}
SCV_LIB=variants/lib_old.so timeout 150 python tools/slab_check.py old 500 8 2>&1 | tail -1
timeout 150 python tools/slab_check.py new 500 8 2>&1 | tail -1
python tools/slab_check.py --cmp old new
SCV_LIB=variants/lib_old.so timeout 150 python tools/slab_check.py old2 959 65 2>&1 | tail -1
timeout 150 python tools/slab_check.py new2 959 65 2>&1 | tail -1
python tools/slab_check.py --cmp old2 new2
rm -f $O/slab_*.npz
run() { SCV_LIB=$2 timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e $3 2>$O/${TAG}_$1.err | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$1 ms/map', round(d['ms_per_step'],1), 'rt', d['roundtrip_rel_err'], 'peak GB', d.get('peak_mem_gb'), 'first map ms', round(d.get('first_map_ms',0))); print({k: round(v,1) for k,v in d['stages_ms_per_step'].items() if v>1})"; }
run base paper_1511_05578_b200/libscurve_b200.so
for f in variants/lib_*.so; do v=$(basename $f .so); [ $v = lib_stats ] || run ${v#lib_} $f; done
run c3_base paper_1511_05578_b200/libscurve_b200.so "--L 512 --jmin 2"
SCV_LIB=variants/lib_stats.so timeout 200 python tools/pipe_stats.py 32 2>&1 | tail -5
