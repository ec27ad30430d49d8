#!/bin/bash
# ncu --set full of the pipelined K=2047 kernels on a beta slab; summaries only come back
# usage: tools/r02_ncu.sh TAG [NB]
TAG=${1:-r02}; NB=${2:-32}
O=gpurun_out; mkdir -p $O /tmp/ncu
timeout 200 python tools/prof_slab.py 1024 $NB > $O/prof_slab_$TAG.log 2>&1 || { cat $O/prof_slab_$TAG.log; exit 1; }
for spec in "k_ana_colgen_p:1:1" "k_pfa_rows_p:2:2" "k_syn_gamma_qp:1:1"; do
  k=${spec%%:*}; rest=${spec#*:}; sk=${rest%%:*}; c=${rest#*:}
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s $sk -c $c -f -o /tmp/ncu/full_${k}_$TAG \
    python tools/prof_slab.py 1024 $NB > $O/ncu_${k}_$TAG.log 2>&1
  { echo "== $k ($TAG, $NB beta rows of L=1024)";
    python tools/ncu_key.py /tmp/ncu/full_${k}_$TAG.ncu-rep;
    python tools/ncu_summary.py /tmp/ncu/full_${k}_$TAG.ncu-rep;
    echo "## per-source-line warp-stall samples (top 40)";
    python tools/ncu_lines.py /tmp/ncu/full_${k}_$TAG.ncu-rep 40; } > $O/ncu_sum_${k}_$TAG.txt 2>&1
done
ls -la $O /tmp/ncu
