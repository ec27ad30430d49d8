#!/bin/bash
# GPU: full gpu suite + smoke, C4 bench (complex, real), C5 streamed, torchrun N=1 sanity.  usage: TAG
TAG=${1:-x}
O=gpurun_out; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> $O/smoke_$TAG.log
timeout 900 python bench.py --steps 3 --warmup 3 > $O/bench_$TAG.log 2>&1; tail -1 $O/bench_$TAG.log > $O/bench_$TAG.json
timeout 600 python bench.py --steps 3 --warmup 3 --real --no-cpu-baseline > $O/bench_real_$TAG.log 2>&1; tail -1 $O/bench_real_$TAG.log > $O/bench_real_$TAG.json
timeout 900 python bench.py --L 2048 --spin 2 --jmin 4 --streamed --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_c5_$TAG.log 2>&1; tail -1 $O/bench_c5_$TAG.log > $O/bench_c5_$TAG.json
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 1 --steps 2 --warmup 3 --no-cpu-baseline > $O/bench_trun_$TAG.log 2>&1; tail -1 $O/bench_trun_$TAG.log > $O/bench_trun_$TAG.json
tail -2 $O/pytest_gpu_$TAG.log; tail -1 $O/smoke_$TAG.log
for f in $O/bench_$TAG.json $O/bench_real_$TAG.json $O/bench_c5_$TAG.json $O/bench_trun_$TAG.json; do python -c "import json; d=json.load(open('$f')); print('$f', round(d['value'],4), round(d['ms_per_step'],1), d.get('roundtrip_rel_err'))" 2>&1 | tail -1; done
