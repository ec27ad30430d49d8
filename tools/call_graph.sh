#!/bin/bash
# GPU: graph replay tests + small-config bench lines with and without --graph.  usage: TAG
TAG=${1:-x}
O=gpurun_out; mkdir -p $O
timeout 600 python -m pytest tests/test_graph.py -m gpu -x -q > $O/pytest_graph_$TAG.log 2>&1; echo "pytest rc=$?" >> $O/pytest_graph_$TAG.log
for cfg in "c1:--L 64 --jmin 2" "c2:--L 128 --spin 2 --jmin 2" "c3:--L 512 --jmin 2"; do
  n=${cfg%%:*}; args=${cfg#*:}
  st=50; [ $n = c3 ] && st=5
  timeout 600 python bench.py $args --steps $st --warmup 3 --graph --no-cpu-baseline > $O/bench_${n}g_$TAG.log 2>&1; tail -1 $O/bench_${n}g_$TAG.log > $O/bench_${n}g_$TAG.json
done
timeout 600 python bench.py --L 64 --jmin 2 --steps 50 --warmup 3 --graph --real --no-cpu-baseline > $O/bench_c1gr_$TAG.log 2>&1; tail -1 $O/bench_c1gr_$TAG.log > $O/bench_c1gr_$TAG.json
tail -3 $O/pytest_graph_$TAG.log
for f in $O/bench_c*g*_$TAG.json; do python -c "import json,sys; d=json.load(open('$f')); print('$f', round(d['value'],2), round(d['ms_per_step'],3), d['gpu_launches'], d['e2e']['value'] if d.get('e2e') else None)" 2>&1 | tail -1; done
