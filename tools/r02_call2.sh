#!/bin/bash
# r02 second GPU pass: the remaining GPU tests + row-engine timing experiments
O=gpurun_out; mkdir -p $O
timeout 2400 python -m pytest tests/test_gpu_parity_full.py tests/test_graph.py tests/test_reference_properties.py tests/test_rotation.py tests/test_sparsity.py tests/test_tiling.py -m gpu -x -q > $O/r02b_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/r02b_pytest_gpu.log
tail -3 $O/r02b_pytest_gpu.log
: > $O/r02b_stage.txt
timeout 120 python tools/stagebench.py 2047 >> $O/r02b_stage.txt 2>&1
for f in variants/lib_*.so; do SCV_LIB=$f timeout 120 python tools/stagebench.py 2047 >> $O/r02b_stage.txt 2>&1; done
cat $O/r02b_stage.txt
