#!/bin/bash
TAG=${1:-x}
O=gpurun_out; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> $O/smoke_$TAG.log
timeout 900 python bench.py --L 2048 --spin 2 --jmin 4 --streamed --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_c5_$TAG.log 2>&1; tail -1 $O/bench_c5_$TAG.log > $O/bench_c5_$TAG.json
tail -2 $O/pytest_gpu_$TAG.log; tail -1 $O/smoke_$TAG.log
python -c "import json; d=json.load(open('$O/bench_c5_$TAG.json')); print(round(d['value'],4), round(d['ms_per_step'],1), d['roundtrip_rel_err'], d['paper_roofline']['frac'], {k: round(v,1) for k,v in d['stages_ms_per_step'].items() if v > 20})"
