#!/bin/bash
# GPU: graph/lane tests + small-config bench lines with --lanes.  usage: TAG
TAG=${1:-x}
O=gpurun_out; mkdir -p $O
timeout 600 python -m pytest tests/test_graph.py -m gpu -x -q > $O/pytest_lanes_$TAG.log 2>&1; echo "pytest rc=$?" >> $O/pytest_lanes_$TAG.log
for cfg in "c1l4:--L 64 --jmin 2 --lanes 4" "c1l8:--L 64 --jmin 2 --lanes 8" "c1l16:--L 64 --jmin 2 --lanes 16" "c2l4:--L 128 --spin 2 --jmin 2 --lanes 4" "c2l8:--L 128 --spin 2 --jmin 2 --lanes 8"; do
  n=${cfg%%:*}; args=${cfg#*:}
  timeout 600 python bench.py $args --steps 20 --warmup 3 --graph --no-cpu-baseline > $O/bench_${n}_$TAG.log 2>&1; tail -1 $O/bench_${n}_$TAG.log > $O/bench_${n}_$TAG.json
done
tail -3 $O/pytest_lanes_$TAG.log
for f in $O/bench_c*l*_$TAG.json; do python -c "import json,sys; d=json.load(open('$f')); print('$f', round(d['value'],2), round(d['ms_per_step'],3), d['gpu_launches'], d['e2e']['value'] if d.get('e2e') else None, d['roundtrip_rel_err'])" 2>&1 | tail -1; done
