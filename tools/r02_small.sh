#!/bin/bash
# small configurations with enough steps to time them (eager, graph, lanes)
O=gpurun_out; mkdir -p $O
run() { timeout 600 python bench.py --no-cpu-baseline $2 > $O/r02v_bench_$1.json 2>$O/r02v_bench_$1.err; python -c "
import json; d=json.loads(open('$O/r02v_bench_$1.json').read().strip().splitlines()[-1]); print('$1', d['config'].get('workload'), round(d['value'],2), d['unit'], round(d['ms_per_step'],3), 'ms rt', d.get('roundtrip_rel_err'), 'launches', d.get('gpu_launches'))" 2>&1 | tail -1; }
run c1 "--L 64 --jmin 2 --steps 300 --warmup 30"
run c1g "--L 64 --jmin 2 --steps 300 --warmup 30 --graph"
run c1l8 "--L 64 --jmin 2 --steps 100 --warmup 10 --graph --lanes 8"
run c2 "--L 128 --spin 2 --jmin 2 --steps 200 --warmup 20"
run c2g "--L 128 --spin 2 --jmin 2 --steps 200 --warmup 20 --graph"
run c2l8 "--L 128 --spin 2 --jmin 2 --steps 100 --warmup 10 --graph --lanes 8"
run c3 "--L 512 --jmin 2 --steps 10 --warmup 3"
run real "--real --steps 5 --warmup 3"
