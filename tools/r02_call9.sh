#!/bin/bash
# r02 GPU pass 9 (re-entry): full GPU suite + default bench + per-role pipeline counters on HEAD
O=gpurun_out; mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -x -q > $O/r02i_pytest_gpu.log 2>&1; tail -3 $O/r02i_pytest_gpu.log
timeout 900 python bench.py > $O/r02i_bench.json 2> $O/r02i_bench.err; tail -c 3000 $O/r02i_bench.json
SCV_LIB=variants/lib_stats.so timeout 200 python tools/pipe_stats.py 32 2>&1 | tail -5
timeout 100 python tools/stagebench.py 2047 | tail -2
