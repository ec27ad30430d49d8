#!/bin/bash
# where the shared-memory bank conflicts of the ring kernels are (per source line)
O=gpurun_out; mkdir -p $O /tmp/ncu; TAG=${1:-r02z}
for spec in "k_pfa_rows_p:2:1" "k_ana_colgen_p:1:1" "k_syn_gamma_qp:1:1"; do
  k=${spec%%:*}; rest=${spec#*:}; sk=${rest%%:*}; c=${rest#*:}
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s $sk -c $c -f -o /tmp/ncu/c_${k} \
    python tools/prof_slab.py 1024 16 > $O/ncu_c_${k}.log 2>&1
  { echo "== $k ($TAG)"; python tools/ncu_conflicts.py /tmp/ncu/c_${k}.ncu-rep 36 --cols; } > $O/${TAG}_conflicts_${k}.txt 2>&1
done
head -45 $O/${TAG}_conflicts_k_pfa_rows_p.txt
