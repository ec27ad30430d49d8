#!/bin/bash
# GPU: new streamed/L>1024 tests + the C5 bench line (1 GPU, streamed)
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "streamed or above_1024 or c5" > $O/pytest_c5.log 2>&1; echo "rc=$?" >> $O/pytest_c5.log
timeout 900 python bench.py --L 2048 --spin 2 --jmin 4 --streamed --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_c5.log 2>&1; tail -1 $O/bench_c5.log > $O/bench_c5.json
timeout 600 python bench.py --streamed --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_c4s.log 2>&1; tail -1 $O/bench_c4s.log > $O/bench_c4s.json
tail -3 $O/pytest_c5.log
