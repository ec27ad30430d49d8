#!/bin/bash
# ncu one k_pfa_rows launch for K=$1 (default 2047); report to gpurun_out/prof_pfa$1.ncu-rep
K=${1:-2047}
python tools/pfa_one.py $K > gpurun_out/p1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_pfa_rows -s 1 -c 1 -o gpurun_out/prof_pfa$K python tools/pfa_one.py $K > gpurun_out/ncu_pfa.log 2>&1
