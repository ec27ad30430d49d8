#!/bin/bash
# GPU-box profiling pass for one build: clean bench line, ncu launch list of
# the bench command, and --set full captures of the L=1024 kernels on a
# 16-row beta slab (tools/prof_slab.py).  usage: tools/profile_round3.sh TAG
TAG=${1:-r01}
O=gpurun_out
mkdir -p $O
python tools/prof_slab.py 1024 16 > $O/prof_slab_$TAG.log 2>&1 || { echo "prof_slab failed"; cat $O/prof_slab_$TAG.log; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_$TAG.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_launch_$TAG.log 2>&1
for spec in "k_ana_colgen_s:1:1" "k_pfa_rows_g:2:2" "k_syn_gamma_q:1:1"; do
  k=${spec%%:*}; rest=${spec#*:}; sk=${rest%%:*}; c=${rest#*:}
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s $sk -c $c -o $O/full_${k}_$TAG \
    python tools/prof_slab.py 1024 16 > $O/ncu_${k}_$TAG.log 2>&1
done
ls $O
