#!/bin/bash
TAG=${1:-x}
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_sparsity.py tests/test_cabi.py -m gpu -x -q > $O/pytest_sp_$TAG.log 2>&1; echo "pytest rc=$?" >> $O/pytest_sp_$TAG.log
timeout 900 python tools/sparsitybench.py 1024 10 > $O/spbench_$TAG.json 2> $O/spbench_$TAG.err
tail -3 $O/pytest_sp_$TAG.log; cut -c1-600 $O/spbench_$TAG.json; tail -3 $O/spbench_$TAG.err
