#!/bin/bash
# GPU: launch list of the L=1024 bench and ncu --set full of the SHT kernels.  usage: TAG
TAG=${1:-x}
O=gpurun_out; mkdir -p $O
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_$TAG.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_launch_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_sht_(bins_w|contract_w)" -s 2 -c 2 -o $O/full_sht_$TAG \
    python tools/sht_prof.py 1024 > $O/ncu_sht_$TAG.log 2>&1
ls $O | grep $TAG
