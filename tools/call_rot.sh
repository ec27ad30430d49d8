#!/bin/bash
# GPU: rotation tests + rotation bench + ncu of the rotation kernels, then the
# v16 profiling pass of the main kernels.  usage: tools/call_rot.sh TAG
TAG=${1:-x}
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_rotation.py tests/test_cabi.py -m gpu -x -q > $O/pytest_rot_$TAG.log 2>&1; echo "pytest rc=$?" >> $O/pytest_rot_$TAG.log
timeout 600 python tools/rotbench.py 1024 5 > $O/rotbench_$TAG.json 2> $O/rotbench_$TAG.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_rot_ -c 2 -o $O/full_rot_$TAG \
    python tools/rotbench.py 512 1 > $O/ncu_rot_$TAG.log 2>&1
bash tools/profile_round3.sh $TAG > $O/profile_$TAG.log 2>&1
tail -3 $O/pytest_rot_$TAG.log; cat $O/rotbench_$TAG.json; tail -3 $O/rotbench_$TAG.err
