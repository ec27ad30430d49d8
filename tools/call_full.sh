#!/bin/bash
# GPU: full gpu test suite, smoke, C4 bench (complex + real), C5 streamed bench.  usage: tools/call_full.sh TAG
TAG=${1:-x}
O=gpurun_out; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> $O/smoke_$TAG.log
timeout 900 python bench.py --steps 3 --warmup 3 > $O/bench_$TAG.log 2>&1; tail -1 $O/bench_$TAG.log > $O/bench_$TAG.json
timeout 600 python bench.py --steps 3 --warmup 3 --real --no-cpu-baseline > $O/bench_real_$TAG.log 2>&1; tail -1 $O/bench_real_$TAG.log > $O/bench_real_$TAG.json
timeout 900 python bench.py --L 2048 --spin 2 --jmin 4 --streamed --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_c5_$TAG.log 2>&1; tail -1 $O/bench_c5_$TAG.log > $O/bench_c5_$TAG.json
tail -2 $O/pytest_gpu_$TAG.log; tail -2 $O/smoke_$TAG.log
