#!/bin/bash
TAG=${1:-x}
O=gpurun_out; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> $O/smoke_$TAG.log
timeout 900 python bench.py --steps 3 --warmup 3 > $O/bench_$TAG.log 2>&1; tail -1 $O/bench_$TAG.log > $O/bench_$TAG.json
timeout 600 python bench.py --steps 3 --warmup 3 --real --no-cpu-baseline > $O/bench_real_$TAG.log 2>&1; tail -1 $O/bench_real_$TAG.log > $O/bench_real_$TAG.json
timeout 600 python bench.py --L 512 --jmin 2 --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_c3_$TAG.log 2>&1; tail -1 $O/bench_c3_$TAG.log > $O/bench_c3_$TAG.json
tail -2 $O/pytest_gpu_$TAG.log; tail -1 $O/smoke_$TAG.log
for f in $O/bench_$TAG.json $O/bench_real_$TAG.json $O/bench_c3_$TAG.json; do python -c "import json; d=json.load(open('$f')); print('$f', round(d['value'],4), round(d['ms_per_step'],2), d['roundtrip_rel_err'], d['e2e']['value'])"; done
