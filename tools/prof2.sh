O=gpurun_out
python tools/prof_slab.py 1024 16 > $O/ps2.log 2>&1
for spec in "k_ana_colgen_s:1:1" "k_syn_gamma_q:1:1"; do
  k=${spec%%:*}; rest=${spec#*:}; sk=${rest%%:*}; c=${rest#*:}
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s $sk -c $c -o $O/full_${k}_r01v11 \
    python tools/prof_slab.py 1024 16 > $O/ncu_${k}_r01v11.log 2>&1
done
ls $O/*.ncu-rep
