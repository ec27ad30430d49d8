#!/bin/bash
# Re-baseline the current HEAD on a GPU box: gpu tests, smoke, bench (complex + real).
O=gpurun_out; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 900 python bench.py --steps 3 --warmup 3 > $O/bench.log 2>&1; tail -1 $O/bench.log > $O/bench.json
timeout 600 python bench.py --steps 3 --warmup 3 --real --no-cpu-baseline > $O/bench_real.log 2>&1; tail -1 $O/bench_real.log > $O/bench_real.json
tail -3 $O/pytest_gpu.log; tail -1 $O/smoke.log
