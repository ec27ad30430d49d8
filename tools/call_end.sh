#!/bin/bash
# GPU: full gpu suite + smoke + rotation bench + C4 bench.  usage: TAG
TAG=${1:-x}
O=gpurun_out; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> $O/smoke_$TAG.log
timeout 600 python tools/rotbench.py 1024 5 > $O/rotbench_$TAG.json 2> $O/rotbench_$TAG.err
timeout 900 python bench.py --steps 3 --warmup 3 > $O/bench_$TAG.log 2>&1; tail -1 $O/bench_$TAG.log > $O/bench_$TAG.json
tail -2 $O/pytest_gpu_$TAG.log; tail -1 $O/smoke_$TAG.log; cut -c1-400 $O/rotbench_$TAG.json
python -c "import json; d=json.load(open('$O/bench_$TAG.json')); print(round(d['value'],4), round(d['ms_per_step'],1), d['roundtrip_rel_err'], d['e2e']['value'], d['clocks'])"
