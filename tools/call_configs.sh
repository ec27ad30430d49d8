#!/bin/bash
# GPU: full gpu suite + smoke, rotation bench, and bench lines at the other BASELINE configs.  usage: TAG
TAG=${1:-x}
O=gpurun_out; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> $O/smoke_$TAG.log
timeout 600 python tools/rotbench.py 1024 5 > $O/rotbench_$TAG.json 2> $O/rotbench_$TAG.err
timeout 600 python bench.py --L 512 --jmin 2 --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_c3_$TAG.log 2>&1; tail -1 $O/bench_c3_$TAG.log > $O/bench_c3_$TAG.json
timeout 600 python bench.py --L 128 --spin 2 --jmin 2 --steps 20 --warmup 3 --no-cpu-baseline > $O/bench_c2_$TAG.log 2>&1; tail -1 $O/bench_c2_$TAG.log > $O/bench_c2_$TAG.json
timeout 600 python bench.py --L 64 --jmin 2 --steps 20 --warmup 3 > $O/bench_c1_$TAG.log 2>&1; tail -1 $O/bench_c1_$TAG.log > $O/bench_c1_$TAG.json
tail -2 $O/pytest_gpu_$TAG.log; tail -1 $O/smoke_$TAG.log; cat $O/rotbench_$TAG.json
